"""Per-layer timing breakdown of traversals (device globaltimer per layer)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1704_02259_b200 as hb

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--uniform", action="store_true")
ap.add_argument("--roots", type=int, default=8)
ap.add_argument("--heuristic", default="beamer")
ap.add_argument("--quiet", action="store_true")
ap.add_argument("--parent-mode", default="minid")
ap.add_argument("--root", type=int, default=-1)
ap.add_argument("--phases", action="store_true")
ap.add_argument("--classes", action="store_true", help="time share per layer class over all roots")
ap.add_argument("--flush", default="write", choices=("write", "read", "none"),
                help="L2 flush before each traversal: write a 256 MB buffer (bench.py's), read it, or none")
a = ap.parse_args()
probs = (0.25,) * 4 if a.uniform else (0.57, 0.19, 0.19, 0.05)
t0 = time.time()
g = hb.generate_graph(hb.GraphParams(scale=a.scale, edgefactor=16, seed=1, probs=probs))
torch.cuda.synchronize()
print(f"graph S{a.scale}: n={g.num_vertices} arcs={g.num_arcs} maxdeg={g.max_degree} wide={g.wide_offsets} build {time.time()-t0:.2f}s", flush=True)
roots = hb.sample_sources(g, 64, 1)[: a.roots] if a.root < 0 else [a.root] * a.roots
p = hb.HeuristicParams(alpha=14, beta=24, heuristic=a.heuristic, counter_mode="edge")
n = g.num_vertices
par = torch.empty(n, dtype=torch.int32, device="cuda"); lev = torch.empty_like(par)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for s in roots[:2]:
    hb.bfs(g, int(s), p, device=True, out=(par, lev), parent_mode=a.parent_mode)
tot = []
cls = {}


def layer_class(x):
    if x.direction == "bottom-up":
        return "BU dense" if x.v_f * 64 >= n else "BU sparse-frontier"
    return "TD hub (e_f>=2^21)" if x.e_f >= 1 << 21 else "TD small"


for s in roots:
    if a.flush == "write":
        flush.fill_(1)
    elif a.flush == "read":
        flush.sum(dtype=torch.int64)
    torch.cuda.synchronize()
    r = hb.bfs(g, int(s), p, device=True, out=(par, lev), parent_mode=a.parent_mode)
    tot.append(r.device_seconds)
    for x in r.trace:
        c = cls.setdefault(layer_class(x), [0.0, 0])
        c[0] += x.elapsed
        c[1] += 1
    c = cls.setdefault("fixed (init, levels, launch)", [0.0, 0])
    c[0] += r.device_seconds - sum(x.elapsed for x in r.trace)
    c[1] += 1
    if not a.quiet:
        lay = " ".join(f"{"B" if x.direction=="bottom-up" else "T"}{x.v_f}[{x.e_f/1e6:.1f}M]:{x.elapsed*1e6:.1f}us" for x in r.trace)
        print(f"root {int(s)}: {r.device_seconds*1e6:.1f}us  sum(layers)={sum(x.elapsed for x in r.trace)*1e6:.1f}us  {lay}", flush=True)
        if a.phases:
            import ctypes as C
            from paper_1704_02259_b200 import _lib
            nl = len(r.trace)
            buf = np.zeros(nl * 8, dtype=np.uint64)
            _lib.check(_lib.load().hbfs_phase_times(g.handle, buf.ctypes.data_as(C.c_void_p), nl))
            kb = np.zeros(1025 * 8, dtype=np.uint64)
            _lib.check(_lib.load().hbfs_phase_times(g.handle, kb.ctypes.data_as(C.c_void_p), 1025))
            k = kb[1024 * 8:1024 * 8 + 8].astype(np.int64)
            print(f"   kernel: init {(k[1]-k[0])/1e3:.1f}us  layers {(k[2]-k[1])/1e3:.1f}us  final-sync {(k[3]-k[2])/1e3:.1f}us  levels {(k[4]-k[3])/1e3:.1f}us")
            dirs = np.array([1 if x.direction == "bottom-up" else 0 for x in r.trace], dtype=np.int32)
            pl = np.zeros(nl, dtype=np.int64)
            _lib.check(_lib.load().hbfs_traversal_bytes_layers(g.handle, int(s), C.c_void_p(lev.data_ptr()),
                       dirs.ctypes.data_as(C.c_void_p), nl, pl.ctypes.data_as(C.c_void_p), None))
            for i, x in enumerate(r.trace):
                t = buf[i * 8:(i + 1) * 8].astype(np.int64)
                print(f"     B_sector {pl[i]/1e6:.1f} MB -> {pl[i]/max(x.elapsed,1e-9)/1e9:.0f} GB/s", end="")
                marks = [(k, t[k] - t[0]) for k in (1, 2, 3, 5, 7, 6, 4) if t[k]]
                print(f"   L{i} {x.direction[0].upper()} v_f={x.v_f} e_f={x.e_f}: " + " ".join(f"s{k}@{v/1e3:.1f}us" for k, v in marks))
m = g.in_edges_total
if a.classes:
    T = sum(tot)
    for k, (t, c) in sorted(cls.items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:30s} {t/len(tot)*1e6:8.1f} us/root  {100*t/T:5.1f}%  ({c} layers)")
print(f"hmean GTEPS {len(tot)*m/sum(tot)/1e9:.2f}  mean us {np.mean(tot)*1e6:.1f}")
