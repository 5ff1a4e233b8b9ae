"""L2 -> DRAM fetch granularity sweep: random-sector probe + S26 traversals per setting.

usage: python tools/l2fetch.py [--scale 26] [--roots 16] [--gran 0,32,64,128]
"""
import argparse, ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1704_02259_b200 as hb
from paper_1704_02259_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--roots", type=int, default=16)
ap.add_argument("--gran", default="-1,32,64,128")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
lib = _lib.load(require_device=True)
prev = C.c_int()
_lib.check(lib.hbfs_l2_fetch_granularity(-1, C.byref(prev)))
print("default L2 fetch granularity:", prev.value, flush=True)
default = prev.value
g = hb.generate_graph(hb.GraphParams(scale=a.scale, edgefactor=16, seed=1))
roots = hb.sample_sources(g, 64, 1)[: a.roots]
p = hb.HeuristicParams(alpha=14, beta=24, heuristic="beamer", counter_mode="edge")
n = g.num_vertices
par = torch.empty(n, dtype=torch.int32, device="cuda"); lev = torch.empty_like(par)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(a.reps):
    for gr in [int(x) for x in a.gran.split(",")]:
        gv = default if gr < 0 else gr
        _lib.check(lib.hbfs_l2_fetch_granularity(gv, None))
        got = C.c_int()
        lib.hbfs_l2_fetch_granularity(-1, C.byref(got))
        rs = {}
        for name, region in (("r256K", 18), ("uni8G", 33)):
            x = C.c_double()
            _lib.check(lib.hbfs_probe_random_sectors(33, region, C.byref(x)))
            rs[name] = round(x.value, 1)
        for s in roots[:2]:
            hb.bfs(g, int(s), p, device=True, out=(par, lev))
        tot = 0.0
        for s in roots:
            flush.fill_(1)
            torch.cuda.synchronize()
            r = hb.bfs(g, int(s), p, device=True, out=(par, lev))
            tot += r.device_seconds
        gteps = len(roots) * g.in_edges_total / tot / 1e9
        print(f"rep {rep} gran set {gv} (reads back {got.value}): probe {rs}  S{a.scale} {a.roots} roots "
              f"{tot/len(roots)*1e3:.3f} ms/root {gteps:.1f} GTEPS", flush=True)
