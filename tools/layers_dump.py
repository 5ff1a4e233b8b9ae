"""Dump every layer of every sampled root (direction, v_f, e_f, device time,
B_sector) as JSON lines, for offline analysis of where the traversal time goes.

usage: python tools/layers_dump.py --scale 26 [--roots 64] [--alpha 14 --beta 24] > layers.jsonl
"""
import argparse, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1704_02259_b200 as hb
from paper_1704_02259_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--uniform", action="store_true")
ap.add_argument("--roots", type=int, default=64)
ap.add_argument("--alpha", type=int, default=14)
ap.add_argument("--beta", type=int, default=24)
ap.add_argument("--heuristic", default="beamer")
a = ap.parse_args()
probs = (0.25,) * 4 if a.uniform else (0.57, 0.19, 0.19, 0.05)
g = hb.generate_graph(hb.GraphParams(scale=a.scale, edgefactor=16, seed=1, probs=probs))
roots = hb.sample_sources(g, 64, 1)[: a.roots]
p = hb.HeuristicParams(alpha=a.alpha, beta=a.beta, heuristic=a.heuristic, counter_mode="edge")
n = g.num_vertices
par = torch.empty(n, dtype=torch.int32, device="cuda")
lev = torch.empty_like(par)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
lib = _lib.load()
for s in roots[:2]:
    hb.bfs(g, int(s), p, device=True, out=(par, lev))
for s in roots:
    flush.fill_(1)
    torch.cuda.synchronize()
    r = hb.bfs(g, int(s), p, device=True, out=(par, lev))
    nl = len(r.trace)
    dirs = np.array([1 if x.direction == "bottom-up" else 0 for x in r.trace], dtype=np.int32)
    pl = np.zeros(nl, dtype=np.int64)
    _lib.check(lib.hbfs_traversal_bytes_layers(g.handle, int(s), C.c_void_p(lev.data_ptr()),
                                               dirs.ctypes.data_as(C.c_void_p), nl,
                                               pl.ctypes.data_as(C.c_void_p), None))
    print(json.dumps({"root": int(s), "total_us": r.device_seconds * 1e6,
                      "layers": [[x.direction[0], x.v_f, x.e_f, x.e_u, round(x.elapsed * 1e6, 1), int(pl[i])]
                                 for i, x in enumerate(r.trace)]}), flush=True)
