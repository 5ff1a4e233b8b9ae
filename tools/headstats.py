"""How many bottom-up candidates does a per-vertex head record resolve?

For every bottom-up layer of a few traversals: candidates (unvisited, degree > 0),
and the share resolved by the first H row entries alone (first frontier hit at a
position < H, or degree <= H and no hit) — the case in which the layer never
touches the row starts or the adjacency array.  Sized the head record of
csrc/graph.cu (`hd`).

usage: python tools/headstats.py [--scale 26] [--roots 4] [--uniform]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1704_02259_b200 as hb

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--roots", type=int, default=4)
ap.add_argument("--uniform", action="store_true")
a = ap.parse_args()
probs = (0.25,) * 4 if a.uniform else (0.57, 0.19, 0.19, 0.05)
g = hb.generate_graph(hb.GraphParams(scale=a.scale, edgefactor=16, seed=1, probs=probs))
n = g.num_vertices
rs = torch.from_numpy(g.row_starts.copy()).cuda()
adj = torch.from_numpy(g.adjacency.copy()).cuda().view(torch.int32)  # ids < 2^31
deg = rs[1:] - rs[:-1]
print(f"n={n} arcs={g.num_arcs} deg>0: {(deg > 0).sum().item()}", flush=True)
p = hb.HeuristicParams(alpha=14, beta=24, heuristic="beamer", counter_mode="edge")
par = torch.empty(n, dtype=torch.int32, device="cuda"); lev = torch.empty_like(par)
HS = (1, 2, 3, 4, 7, 8)
for s in hb.sample_sources(g, 64, 1)[: a.roots]:
    r = hb.bfs(g, int(s), p, device=True, out=(par, lev))
    print(f"root {int(s)}: " + " ".join(f"{'B' if x.direction == 'bottom-up' else 'T'}{x.v_f}" for x in r.trace))
    for x in r.trace:
        if x.direction != "bottom-up":
            continue
        L = x.layer - 1
        c = torch.nonzero(((lev > L) | (lev < 0)) & (deg > 0)).squeeze(1)
        dc, sc = deg[c], rs[c]
        first = torch.full_like(dc, 1 << 40)
        for j in reversed(range(max(HS))):
            ok = dc > j
            idx = torch.where(ok, sc + j, torch.zeros_like(sc))
            hit = ok & (lev[adj[idx].long()] == L)
            first = torch.where(hit, torch.full_like(first, j), first)
        out = [f"L{L} cand {len(c)} found-in-{max(HS)} {(first < (1 << 40)).sum().item()}"]
        for H in HS:
            res = (first < H) | (dc <= H)
            out.append(f"H{H}:{res.float().mean().item() * 100:.1f}%")
        print("   " + " ".join(out), flush=True)
