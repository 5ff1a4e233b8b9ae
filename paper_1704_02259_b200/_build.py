"""Build libhbfs.so in-tree: nvcc for sm_100a, all of csrc/*.cu in one shared library.

The library is the product (the C ABI declared in include/hbfs.h); it is built
here on the CPU box (nvcc cross-compiles) and travels to the GPU box with the
repo snapshot.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(CSRC, "libhbfs.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [*__import__("shlex").split(__import__("os").environ.get("HBFS_NVCC_EXTRA", "")), "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(REPO, "include", "hbfs.h")]


def needs_build() -> bool:
    return _stale(LIB) or _stale(LIB_CHECKED)


# The bounds-checked variant (device index checks, HB_DCHECK) that
# tools/sanitize.py and tests/test_gpu_sanitize.py run in place of
# compute-sanitizer, which the GPU pool does not allow.
LIB_CHECKED = os.path.join(CSRC, "libhbfs_checked.so")
VARIANTS = {LIB: ("build", []), LIB_CHECKED: ("build_checked", ["-DHBFS_CHECKED"])}


def _stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    """Build libhbfs.so and libhbfs_checked.so (objects compiled in parallel)."""
    jobs = []
    for lib, (sub, extra) in VARIANTS.items():
        if not force and not _stale(lib):
            continue
        objdir = os.path.join(CSRC, sub)
        os.makedirs(objdir, exist_ok=True)
        objs = []
        procs = []
        for src in sources():
            obj = os.path.join(objdir, os.path.basename(src) + ".o")
            objs.append(obj)
            if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(
                os.path.getmtime(p) for p in [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(REPO, "include", "hbfs.h")]
            ):
                continue
            cmd = [NVCC, *ARCH, *FLAGS, *extra, "-I", os.path.join(REPO, "include"), "-c", src, "-o", obj]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        jobs.append((lib, objs, procs))
    for lib, objs, procs in jobs:
        for src, p in procs:
            out, _ = p.communicate()
            if p.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src}:\n{out[-6000:]}")
            if verbose and out:
                print(out)
        tmp = lib + ".tmp"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, lib)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
