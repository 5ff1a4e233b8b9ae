"""Build an experiment variant of libhbfs.so: csrc/ with bfs.cu replaced by
the given file, linked to the given output path (A/B runs via HBFS_LIB)."""
import os
import shutil
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_02259_b200 import _build as B  # noqa: E402


def main(bfs_src, out):
    d = tempfile.mkdtemp()
    objs = []
    procs = []
    for src in B.sources():
        if os.path.basename(src) == "bfs.cu":
            src2 = os.path.join(d, "bfs.cu")
            shutil.copy(bfs_src, src2)
            src = src2
        obj = os.path.join(d, os.path.basename(src) + ".o")
        objs.append(obj)
        extra = os.environ.get("HBFS_VAR_FLAGS", "").split()  # e.g. -DHBFS_KBLOCK=384
        cmd = [B.NVCC, *B.ARCH, *B.FLAGS, *extra, "-I", os.path.join(B.REPO, "include"), "-I", B.CSRC, "-c", src, "-o", obj]
        procs.append(subprocess.Popen(cmd))
    for p in procs:
        assert p.wait() == 0
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", out, *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"], check=True)
    print(out)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
