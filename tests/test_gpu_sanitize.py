"""Memory-safety evidence without compute-sanitizer (closed on the GPU pool):
tools/sanitize.py — every kernel family at SCALE 12 with the column-blocked,
harvest, deferred-level and multi-launch paths forced, results checked against
the C oracle — runs on the bounds-checked build (device index checks) with
guard bands behind every device buffer; both must stay clean."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("lib", ["libhbfs_checked.so", "libhbfs.so"])
def test_sanitize_workload_guards_and_index_checks(cuda, lib):
    path = os.path.join(REPO, "paper_1704_02259_b200", "csrc", lib)
    assert os.path.exists(path), f"{lib} must be built (paper_1704_02259_b200/_build.py)"
    env = {**os.environ, "HBFS_GUARD": "1", "HBFS_LIB": path}
    r = subprocess.run([sys.executable, os.path.join(REPO, "tools", "sanitize.py")], env=env,
                       capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "sanitize workload ok" in out
    assert "guards on" in out and "0 clobbered" in out
    if lib == "libhbfs_checked.so":
        assert "index checks on: flags 0x0" in out
