"""Timing of the 1D-partitioned path (mgpu.DistBfs + csrc/part.cu) on ONE GPU
with P logical ranks (LocalComm: the ranks' kernels run one after another, so
the time is the sum over ranks = the work of the slowest-rank bound times P).
Shows per-rank kernel efficiency against the single-GPU persistent kernel."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1704_02259_b200 as hb
from paper_1704_02259_b200.mgpu import CudaRankOps, DistBfs, LocalComm, LocalPersistBfs, NcclBfs

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--roots", type=int, default=8)
ap.add_argument("--ranks", default="1,2,4")
ap.add_argument("--layers", action="store_true")
ap.add_argument("--persist", action="store_true", help="P ranks through the persistent partition kernel (C++ loop)")
a = ap.parse_args()
params = hb.GraphParams(scale=a.scale, edgefactor=16, seed=1)
g = hb.generate_graph(params)
roots = hb.sample_sources(g, a.roots, 1)
p = hb.HeuristicParams(alpha=14, beta=24, heuristic="beamer", counter_mode="edge")
m = g.in_edges_total
t = []
for s in roots:
    r = hb.bfs(g, int(s), p, device=True)
    t.append(r.device_seconds)
print(f"S{a.scale} single-GPU persistent kernel: hmean {len(t) * m / sum(t) / 1e9:.2f} GTEPS, mean {np.mean(t) * 1e3:.3f} ms")
ref = {int(s): hb.bfs(g, int(s), p, device=False) for s in roots[:2]}
g.free()
for P in [int(x) for x in a.ranks.split(",")]:
    ranks = [CudaRankOps.generate(params, P, r) for r in range(P)]
    db = LocalPersistBfs(ranks) if a.persist else DistBfs(ranks, LocalComm(P))
    db.bfs(int(roots[0]), p)
    ts = []
    for s in roots:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = db.bfs(int(s), p)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        if int(s) in ref:
            par = np.concatenate([o[0] for o in db.outputs()])
            lev = np.concatenate([o[1] for o in db.outputs()])
            assert np.array_equal(lev, ref[int(s)].level) and np.array_equal(par, ref[int(s)].parent), "mismatch"
        if a.layers and s == roots[0]:
            print("   " + " ".join(f"{'B' if x.direction == 'bottom-up' else 'T'}{x.v_f}:{x.elapsed * 1e3:.2f}ms" for x in res.trace))
    print(f"P={P} logical ranks on one GPU: hmean {len(ts) * m / sum(ts) / 1e9:.2f} GTEPS (sum over ranks), "
          f"mean {np.mean(ts) * 1e3:.3f} ms per root = {np.mean(ts) / P * 1e3:.3f} ms per rank-share")
    for r in ranks:
        r.free()

# the C++ loop over NCCL, one rank (the per-layer host cost without Python)
ops = CudaRankOps.generate(params, 1, 0)
nb = NcclBfs(ops, 1, 0)
nb.bfs(int(roots[0]), p)
ts = []
for s in roots:
    res = nb.bfs(int(s), p)
    ts.append(res.seconds)
    if s == roots[0] and a.layers:
        print("   layers: " + " ".join(f"{'B' if x.direction == 'bottom-up' else 'T'}{x.v_f}" for x in res.trace))
    if int(s) in ref:
        par, lev = nb.outputs()[0]
        assert np.array_equal(lev, ref[int(s)].level) and np.array_equal(par, ref[int(s)].parent), "mismatch"
print(f"NCCL C++ loop, world 1: hmean {len(ts) * m / sum(ts) / 1e9:.2f} GTEPS, mean {np.mean(ts) * 1e3:.3f} ms per root")
nb.free()
ops.free()
