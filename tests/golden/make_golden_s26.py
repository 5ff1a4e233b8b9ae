"""Golden digests for the headline graph, Kronecker SCALE 26 (BASELINE config 4),
from the REFERENCE's own code paths (build container only):

* the CSR built by the C oracle's generator + csr_build (oracle/hbfs_oracle.c) —
  the graph `bench.py --impl reference` traverses — as SHA-256 of the int64
  row_starts and uint32 adjacency.  The GPU test asserts the device-built CSR
  has the same digests, so both bench arms provably run on one graph.
  (The reference's numpy generate() refuses SCALE 26 without an edge budget
  and needs > 60 GB here; the C restatement is pinned bit-exact against it
  at C1/C2/C3 and SCALE 24, hashes.json / hashes_s24.json.)
* the 64 roots of the reference's harness.sample_sources on that graph;
* for the first ROOTS roots: levels from the reference's engine.bfs_reference
  (compiled _native, FIFO parents digest too) and the parents + trace of the
  reference's stock hybrid_bfs(alpha=14, beta=24, use_simd=True, native engine).

Usage: python tests/golden/make_golden_s26.py [roots]   (~10 min, ~40 GB RAM)
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as MG  # noqa: E402  (loads the reference read-only)

from hybfs import csr, engine, harness  # noqa: E402

from oracle import oracle as O  # noqa: E402

ROOTS = 8


def main():
    nroots = int(sys.argv[1]) if len(sys.argv) > 1 else ROOTS
    t0 = time.time()
    O.build()
    u, v = O.generate(26, 16, 1)
    rec = {"params": {"scale": 26, "edgefactor": 16, "seed": 1, "probs": [0.57, 0.19, 0.19, 0.05]},
           "u_sha": MG.sha(u), "v_sha": MG.sha(v)}
    h = O.csr_build(u, v, 1 << 26)
    del u, v
    print(f"oracle generate + csr_build: {time.time() - t0:.1f}s", flush=True)
    g = csr.CsrGraph(num_vertices=h.num_vertices, num_arcs=int(h.row_starts[-1]),
                     row_starts=h.row_starts, adjacency=h.adjacency, in_edges_total=h.in_edges_total)
    rec.update({"n": g.num_vertices, "arcs": g.num_arcs, "m": g.in_edges_total,
                "rs_sha": MG.sha(g.row_starts), "adj_sha": MG.sha(g.adjacency)})
    srcs = harness.sample_sources(g, 64, 1)
    rec["sources"] = [int(x) for x in srcs]
    rec["roots"] = {}
    for s in srcs[:nroots]:
        t1 = time.time()
        tree, lev = engine.bfs_reference(g, int(s), engine="native")
        r = {"level_sha": MG.sha(lev), "fifo_parent_sha": MG.sha(tree.parent),
             "reached": int((lev >= 0).sum()), "depth": int(lev.max())}
        par, tr = MG.run_mode(g, s, "simd_a14b24")
        r["simd_a14b24"] = {"parent_sha": MG.sha(par), "trace": tr}
        rec["roots"][str(int(s))] = r
        print(f"root {int(s)}: {time.time() - t1:.1f}s", flush=True)
    with open(os.path.join(HERE, "hashes_s26.json"), "w") as fh:
        json.dump({"S26_kron": rec}, fh, indent=1)
    print(f"wrote hashes_s26.json in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
