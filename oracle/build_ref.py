"""TEST INFRASTRUCTURE — recipe that compiles the reference's own native kernels.

Compiles ``/root/reference/pkg/src/hybfs/_native.pyx`` (+ ``bu_probe.h``) where it
lies, with Cython + gcc, into ``oracle/_ref/<variant>/hybfs/_native*.so``.  Nothing
from the reference is copied into the repo: the generated C and object files go to
a scratch dir under /tmp and only the built extension lands in ``oracle/_ref/``
(git-ignored, but NOT gpurun-ignored, so it travels to the GPU box).

Two variants are built because the GPU box's host CPU is not known here:

* ``avx512`` — ``-O3 -march=x86-64-v4``: the reference's AVX-512 masked
  gather/scatter probe (``bu_probe.h:18-64``) is compiled in.  The reference's own
  flags are ``-O3 -march=native`` (``setup.py:11``); x86-64-v4 is the portable
  spelling of the AVX-512F/BW/CD/DQ/VL subset the probe needs.
* ``scalar`` — ``-O3 -march=x86-64-v2``: ``__AVX512F__`` undefined, so the
  reference's scalar twin (``bu_probe.h:66-106``) is compiled in.

``oracle.refnative.load()`` picks the variant the running CPU supports.
Only ``tests/``, ``bench.py --impl reference`` / ``cpu_baseline`` and
``__graft_entry__`` use this.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import sysconfig
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src/hybfs"
OUT_ROOT = os.path.join(HERE, "_ref")
VARIANTS = {
    "avx512": ["-O3", "-march=x86-64-v4"],
    "scalar": ["-O3", "-march=x86-64-v2"],
}


def _ext_suffix() -> str:
    return sysconfig.get_config_var("EXT_SUFFIX") or ".so"


def built_paths() -> dict:
    return {
        v: os.path.join(OUT_ROOT, v, "hybfs", "_native" + _ext_suffix())
        for v in VARIANTS
    }


def install_package(quiet: bool = True) -> None:
    """Ship the reference's stock Python package next to each compiled _native:
    the unmodified ``hybfs/*.py`` of /root/reference land in
    ``oracle/_ref/<variant>/hybfs/`` (git-ignored build output, like the .so),
    so the GPU box can import the stock ``hybfs`` — its controller
    (``hybrid.hybrid_bfs``), engine dispatch and harness — for the bench's
    reference arm and the reference-side integration tests
    (``oracle.refpkg``).  Files are copied verbatim and never edited."""
    for variant in VARIANTS:
        dst = os.path.join(OUT_ROOT, variant, "hybfs")
        os.makedirs(dst, exist_ok=True)
        for name in sorted(os.listdir(REF_SRC)):
            if not name.endswith(".py"):
                continue
            src = os.path.join(REF_SRC, name)
            out = os.path.join(dst, name)
            if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
                shutil.copyfile(src, out)
        if not quiet:
            print(f"stock hybfs package ({variant}) -> {dst}")


def build(force: bool = False, quiet: bool = True) -> dict:
    """Build both variants if the reference sources are present; return paths."""
    paths = built_paths()
    if not os.path.isdir(REF_SRC):
        return {v: p for v, p in paths.items() if os.path.exists(p)}
    install_package(quiet)
    pyx = os.path.join(REF_SRC, "_native.pyx")
    hdr = os.path.join(REF_SRC, "bu_probe.h")
    src_mtime = max(os.path.getmtime(pyx), os.path.getmtime(hdr))
    import numpy as np
    from Cython.Compiler.Main import compile_single, CompilationOptions, default_options

    with tempfile.TemporaryDirectory(prefix="hbfs_ref_") as tmp:
        c_file = os.path.join(tmp, "_native.c")
        need = force or any(
            not os.path.exists(p) or os.path.getmtime(p) < src_mtime for p in paths.values()
        )
        if not need:
            return paths
        opts = CompilationOptions(default_options)
        opts.language_level = 3
        opts.output_file = c_file
        # Module name must be hybfs._native (the pyx is compiled as part of
        # the hybfs package in the reference's setup.py).
        res = compile_single(pyx, opts, full_module_name="hybfs._native")
        if res.num_errors:
            raise RuntimeError("cython failed on the reference _native.pyx")
        inc = [
            np.get_include(),
            REF_SRC,
            sysconfig.get_paths()["include"],
        ]
        for variant, flags in VARIANTS.items():
            out = paths[variant]
            os.makedirs(os.path.dirname(out), exist_ok=True)
            cmd = (
                ["gcc", "-shared", "-fPIC", "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION"]
                + flags
                + [f"-I{d}" for d in inc]
                + [c_file, "-o", out + ".tmp"]
            )
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"gcc failed for {variant}:\n{r.stderr[-4000:]}")
            os.replace(out + ".tmp", out)
            if not quiet:
                print(f"built reference _native ({variant}) -> {out}")
    return paths


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, quiet=False)
    print(p)
