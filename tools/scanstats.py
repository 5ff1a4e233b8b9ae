"""Scan statistics of one bottom-up layer (experiment tool): candidates,
entries probed, rows left for the warp-cooperative tail after the lane phase."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1704_02259_b200 as hb

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--root", type=int, required=True)
ap.add_argument("--layer", type=int, required=True, help="frontier level of the BU layer")
ap.add_argument("--lane-entries", type=int, default=16)
a = ap.parse_args()
g = hb.generate_graph(hb.GraphParams(scale=a.scale, edgefactor=16, seed=1))
p = hb.HeuristicParams(alpha=14, beta=24, heuristic="beamer", counter_mode="edge")
r = hb.bfs(g, a.root, p, device=True)
lev = r.level.long()
rs = torch.from_numpy(np.asarray(g.row_starts)).cuda()
adj = torch.from_numpy(np.asarray(g.adjacency).view(np.int32)).cuda()
n = g.num_vertices
deg = rs[1:] - rs[:-1]
L = a.layer
front = lev == L
cand = ((lev > L) | (lev < 0)) & (deg > 0)
print(f"frontier {int(front.sum())}  candidates {int(cand.sum())}  deg-sum(cand) {int(deg[cand].sum())}")
first = torch.full((n,), 1 << 40, dtype=torch.int64, device="cuda")
CH = 1 << 28
for c0 in range(0, adj.numel(), CH):
    c1 = min(adj.numel(), c0 + CH)
    idx = torch.arange(c0, c1, device="cuda")
    hit = front[adj[c0:c1].long()]
    rows = torch.searchsorted(rs, idx, right=True) - 1
    pos = torch.where(hit, idx - rs[rows], torch.full_like(idx, 1 << 40))
    first.scatter_reduce_(0, rows, pos, reduce="amin")
found = cand & (first < (1 << 40))
scan = torch.where(found, first + 1, deg)[cand]
print(f"found {int(found.sum())}  entries probed (to first hit or row end) {int(scan.sum())}")
fp = first[found]
tot = float(found.sum())
print("first-hit position among found: " + ", ".join(
    f"{k}: {100 * float((fp == k).sum()) / tot:.1f}%" for k in range(4)) +
      f", >=4: {100 * float((fp >= 4).sum()) / tot:.1f}%")
# probes issued by the current lane phase: whole aligned vectors until the hit / row end
off_all = (rs[:-1] & 3)
vec_probes = torch.minimum(((off_all + torch.where(found, first + 1, deg) + 3) // 4) * 4 - off_all, deg)[cand]
print(f"probes with 4-entry vectors {int(vec_probes.sum())}  vs exact {int(scan.sum())}")
# lane phase covers the aligned vectors starting at rs & ~3: entries up to LE - (rs & 3)
off = (rs[:-1] & 3)[cand]
lane_cov = (a.lane_entries - off).clamp(min=0)
tail = scan > lane_cov
tl = (scan - lane_cov).clamp(min=0)[tail]
print(f"tail rows {int(tail.sum())} ({100*float(tail.float().mean()):.1f}% of candidates)  tail entries {int(tl.sum())}")
q = torch.quantile(tl.float()[:1 << 24], torch.tensor([0.5, 0.9, 0.99], device="cuda"))
print(f"tail length p50/p90/p99 {q.tolist()}  steps of 128: {int(((tl + 127) // 128).sum())}")
# entries probed per candidate, bucketed (where the layer's probe work sits)
edges = [0, 4, 8, 16, 32, 128, 1024, 1 << 40]
sc = scan
for lo_, hi_ in zip(edges[:-1], edges[1:]):
    msk = (sc > lo_) & (sc <= hi_)
    print(f"  scan ({lo_:>5},{hi_ if hi_ < 1 << 40 else 'inf':>5}]: rows {int(msk.sum()):>10}  entries {int(sc[msk].sum()):>12}")
