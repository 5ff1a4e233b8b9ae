"""TEST INFRASTRUCTURE — loader for the reference's compiled ``hybfs._native``.

Loads the extension built by ``oracle/build_ref.py`` (AVX-512 variant when the
host CPU has AVX-512F, else the scalar variant) under its own module name
``hybfs._native``.  The module exposes the reference's native layer kernels
(``_native.pyx:39-239``): ``bfs_reference``, ``top_down_layer``,
``bottom_up_layer``, ``bottom_up_multiple_set``, ``top_down_chunked``,
``probe_uses_simd``.

Only tests, golden generation and the bench's reference arm may import this.
"""

from __future__ import annotations

import importlib.machinery
import importlib.util
import os
import sys

from . import build_ref


def cpu_has_avx512f() -> bool:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("flags"):
                    return " avx512f " in (line.rstrip() + " ")
    except OSError:
        pass
    return False


_MOD = None


def load():
    """Return the reference ``_native`` module, or None if it was never built."""
    global _MOD
    if _MOD is not None:
        return _MOD
    if "hybfs._native" in sys.modules:
        _MOD = sys.modules["hybfs._native"]
        return _MOD
    paths = build_ref.built_paths()
    order = ["avx512", "scalar"] if cpu_has_avx512f() else ["scalar"]
    for variant in order:
        p = paths[variant]
        if not os.path.exists(p):
            continue
        loader = importlib.machinery.ExtensionFileLoader("hybfs._native", p)
        spec = importlib.util.spec_from_file_location("hybfs._native", p, loader=loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        sys.modules["hybfs._native"] = mod
        mod.__variant__ = variant
        _MOD = mod
        return mod
    return None
