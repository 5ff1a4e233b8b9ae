"""Per-rank cost of the P-rank partitioned traversal, emulated on ONE GPU.

All P ranks of the partition live on this GPU and run through the same C++
loop as the multi-GPU path (hbfs_mgl_bfs: the persistent kernel per rank and
layer, exchanges as device copies), one rank after another; so the measured
time is the SUM of the ranks' compute, and sum / P is what one GPU of a P-GPU
run spends computing (the NVLink exchange time is not included).  Levels and
parents are checked against the single-GPU traversal of the same graph.

  python tools/mgpu_project.py --scale 28 --ranks 8 --roots 8
"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1704_02259_b200 as hb
from paper_1704_02259_b200.mgpu import CudaRankOps, LocalPersistBfs

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--ranks", type=int, default=8)
ap.add_argument("--roots", type=int, default=8)
a = ap.parse_args()
params = hb.GraphParams(scale=a.scale, edgefactor=16, seed=1)
p = hb.HeuristicParams(alpha=14, beta=24, heuristic="beamer", counter_mode="edge")
g = hb.generate_graph(params)
roots = [int(x) for x in hb.sample_sources(g, a.roots, 1)]
ref, t1 = {}, []
for s in roots:
    r = hb.bfs(g, s, p, device=False)
    ref[s] = (r.level, r.parent)
    t1.append(r.device_seconds)
g.free()
del g
torch.cuda.empty_cache()
m = params.num_edges
print(f"S{a.scale} one GPU (persistent kernel): hmean {len(t1) * m / sum(t1) / 1e9:.1f} GTEPS, "
      f"mean {np.mean(t1) * 1e3:.3f} ms", flush=True)
ranks = [CudaRankOps.generate(params, a.ranks, r) for r in range(a.ranks)]
lb = LocalPersistBfs(ranks)
lb.bfs(roots[0], p)
ts = []
for s in roots:
    res = lb.bfs(s, p)
    ts.append(res.seconds)
    print(f"  root {s}: {res.seconds * 1e3:.3f} ms summed over ranks: " + " ".join(
        f"{'B' if x.direction == 'bottom-up' else 'T'}{x.v_f}:{x.elapsed * 1e3:.2f}" for x in res.trace), flush=True)
    outs = lb.outputs()
    lev = np.concatenate([o[1] for o in outs])
    par = np.concatenate([o[0] for o in outs])
    assert np.array_equal(lev, ref[s][0]) and np.array_equal(par, ref[s][1]), f"mismatch at root {s}"
share = np.mean(ts) / a.ranks
print(f"P={a.ranks} ranks emulated on one GPU: sum over ranks {np.mean(ts) * 1e3:.3f} ms per traversal, "
      f"per-rank share {share * 1e3:.3f} ms -> {m / share / 1e9:.0f} GTEPS of compute per {a.ranks}-GPU traversal "
      f"(exchange time not included); all {len(roots)} roots bit-exact vs one GPU", flush=True)
