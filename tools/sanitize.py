"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every kernel family of libhbfs.so at SCALE <= 14, each checked against the C
oracle so a run that "passes" the sanitizer also computed the right answer.

compute-sanitizer is closed on the GPU pool (runs under it left GPUs needing
a reset), so the same workload runs with the library's own checks instead:

  HBFS_GUARD=1 HBFS_LIB=paper_1704_02259_b200/csrc/libhbfs_checked.so \
      python tools/sanitize.py

* HBFS_GUARD=1: a guard band behind every device buffer, verified after each
  section (hbfs_debug_guards) — out-of-bounds writes;
* libhbfs_checked.so (-DHBFS_CHECKED): device index checks on the traversal
  kernels' queue / chunk-start / parent / level / adjacency / row-start /
  level-pass indices (hbfs_debug_checks) — out-of-bounds reads and writes;
* every result compared with the C oracle — races that lose updates.

Covers: device generator + CSR build (keep-dup, dedup, source-range pieces),
source sampling, the persistent traversal kernel in every mode (reference /
Beamer, scalar / simd, forced directions, min-id and any parents), with the
column-blocked, harvest and deferred-level paths forced on, the large-graph
kernel variant, multi-launch resume, the per-layer kernels, the FIFO
reference BFS, the validator and byte accounting, and the partition kernels
(P = 2, one process).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true", help="fewer roots/modes (racecheck is slow)")
ap.add_argument("--scale", type=int, default=12)
a = ap.parse_args()

# knobs read when a graph's workspace is created: force the large-graph paths
os.environ.setdefault("HBFS_CB_MIN_N", "0")
os.environ.setdefault("HBFS_CB_MIN_ARCS", "0")
os.environ.setdefault("HBFS_CB_RANGES", "5")
os.environ.setdefault("HBFS_HARVEST_MIN_ARCS", "4096")
os.environ.setdefault("HBFS_DEFER_LEVELS_MIN_N", "0")

import paper_1704_02259_b200 as hb  # noqa: E402
from oracle import oracle as O  # noqa: E402

O.build()
checks = 0


def check(ok, what):
    global checks
    if not ok:
        raise SystemExit(f"MISMATCH: {what}")
    checks += 1


def debug_state(section):
    """Guard bands and device index-check flags after a section."""
    import ctypes as C

    from paper_1704_02259_b200 import _lib

    lib = _lib.load()
    en, nchk, nbad, first = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
    _lib.check(lib.hbfs_debug_guards(C.byref(en), C.byref(nchk), C.byref(nbad), C.byref(first)))
    flags, is_checked = C.c_uint32(), C.c_int()
    _lib.check(lib.hbfs_debug_checks(C.byref(flags), 0, C.byref(is_checked)))
    print(f"[{section}] guards {'on' if en.value else 'off'}: {nchk.value} bands checked, "
          f"{nbad.value} clobbered; index checks {'on' if is_checked.value else 'off'}: "
          f"flags 0x{flags.value:x}", flush=True)
    if nbad.value:
        raise SystemExit(f"GUARD CLOBBERED after {section}: first buffer of {first.value} bytes")
    if flags.value:
        raise SystemExit(f"INDEX CHECK FAILED after {section}: flags 0x{flags.value:x}")


params = hb.GraphParams(scale=a.scale, edgefactor=16, seed=1)
g = hb.generate_graph(params)
u, v = O.generate(a.scale, 16, 1)
host = O.csr_build(u, v, 1 << a.scale)
check(np.array_equal(g.row_starts, host.row_starts) and np.array_equal(g.adjacency, host.adjacency), "csr")
gd = hb.generate_graph(params, dedup=True)
hd = O.csr_build(u, v, 1 << a.scale, dedup=True)
check(np.array_equal(gd.adjacency, hd.adjacency), "dedup csr")
gd.free()
os.environ["HBFS_BUILD_PIECES"] = "3"
gp = hb.from_arrays(u, v, 1 << a.scale)
del os.environ["HBFS_BUILD_PIECES"]
check(np.array_equal(gp.adjacency, host.adjacency), "pieces csr")
gp.free()
roots = hb.sample_sources(g, 8, 1)
check(np.array_equal(roots, O.sample_sources(host, 8, 1)), "roots")
roots = roots[:3] if a.quick else roots
debug_state("generator + CSR build + sampling")

modes = [dict(use_simd=True), dict(use_simd=False), dict(use_simd=True, force_direction="bottom-up"),
         dict(use_simd=False, force_direction="top-down")]
beamer = dict(heuristic="beamer", counter_mode="edge", alpha=14, beta=24)
for variant in ("4", "3"):  # small-graph and large-graph kernel variants
    os.environ["HBFS_KERNEL_VARIANT"] = variant
    gv = hb.generate_graph(params)
    for s in roots:
        s = int(s)
        _, lev = O.bfs_reference(host, s)
        for kw in (modes[:2] if a.quick else modes):
            r = hb.bfs(gv, s, device=False, **kw)
            par, lev2, _ = O.hybrid_bfs(host, s, **kw)
            check(np.array_equal(r.level, lev) and np.array_equal(r.parent, par), f"bfs {variant} {s} {kw}")
        r = hb.bfs(gv, s, hb.HeuristicParams(**beamer), device=False)
        par, _, _ = O.hybrid_bfs(host, s, use_simd=True, **beamer)
        check(np.array_equal(r.parent, par), f"beamer {s}")
        r = hb.bfs(gv, s, device=False, parent_mode="any", force_direction="top-down")
        check(np.array_equal(r.level, lev) and O.validate_tree(host, s, r.parent)[0] == 0, f"any {s}")
        rep = hb.validate_tree(gv, s, r.parent, r.level)
        check(rep.ok, f"validator {s}")
        rd = hb.bfs(gv, s, device=True)
        bs, bu = hb.traversal_bytes(gv, s, rd.level, rd.trace)
        check(bs > 0 and bu > 0, "bytes")
    debug_state(f"traversals, kernel variant {variant}")
    gv.free()
os.environ.pop("HBFS_KERNEL_VARIANT")

# multi-launch resume (> 1024 layers) on a path
n = 1500
gpath = hb.from_arrays(np.arange(n - 1, dtype=np.uint32), np.arange(1, n, dtype=np.uint32), n)
r = hb.bfs(gpath, 0, device=False)
check(np.array_equal(r.level, np.arange(n, dtype=np.int32)), "deep path")
debug_state("multi-launch resume")

# per-layer kernels (the _native surface) and the FIFO reference BFS
from paper_1704_02259_b200 import native  # noqa: E402

s = int(roots[0])
fp, fl = native.bfs_reference(host.row_starts, host.adjacency, host.num_vertices, s)
rp, rl = O.bfs_reference(host, s)
check(np.array_equal(fl, rl) and np.array_equal(fp, rp), "fifo reference")
nw = (host.num_vertices + 31) // 32
for layer_fn in ("top_down_chunked", "bottom_up_multiple_set", "bottom_up_layer"):
    inw = np.zeros(nw, np.uint32)
    vis = np.zeros(nw, np.uint32)
    out = np.zeros(nw, np.uint32)
    inw[s >> 5] = vis[s >> 5] = np.uint32(1 << (s & 31))
    par = np.full(host.num_vertices, 0xFFFFFFFF, np.uint32)
    par[s] = s
    args = (host.row_starts, host.adjacency, inw, vis, out, par, host.num_vertices)
    if layer_fn == "bottom_up_multiple_set":
        getattr(native, layer_fn)(*args, 8, None, np.zeros(nw, np.uint32), np.zeros(nw, np.uint32))
    else:
        getattr(native, layer_fn)(*args)
    check(int(np.bitwise_count(out).sum()) == int(((rl == 1)).sum()), f"layer {layer_fn}")
debug_state("per-layer kernels + FIFO reference")

# partition kernels, P = 2 in one process (no kernel waits on another)
from paper_1704_02259_b200.mgpu import CudaRankOps, DistBfs, LocalComm, LocalPersistBfs  # noqa: E402

ranks = [CudaRankOps.from_csr(host.row_starts, host.adjacency, host.in_edges_total, 2, r) for r in range(2)]
for db in (DistBfs(ranks, LocalComm(2)), LocalPersistBfs(ranks)):
    for s in roots[:2]:
        s = int(s)
        db.bfs(s, hb.HeuristicParams(**beamer), use_simd=True)
        outs = db.outputs()
        lev = np.concatenate([o[1] for o in outs])
        check(np.array_equal(lev, O.bfs_reference(host, s)[1]), f"partition {type(db).__name__} {s}")
debug_state("partition kernels")
print(f"sanitize workload ok: {checks} checks")
