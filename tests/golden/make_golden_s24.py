"""Golden digests for a Kronecker SCALE 24 graph from the REFERENCE itself
(build container only): the large-graph kernel variant (n >= 2^24: column-
blocked / harvest top-down, deferred level stamping, 2 CTAs/SM) is pinned at
a size the reference can still build here.  Writes hashes_s24.json with the
keep-dup and dedup CSR digests, the 64 sampled roots, and for 4 roots the
levels (engine.bfs_reference), the FIFO parents of _native.bfs_reference and
the parents + trace of hybrid_bfs(alpha=14, beta=24, native engine).

Usage: python tests/golden/make_golden_s24.py   (~10 min, ~20 GB RAM)
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as MG  # noqa: E402  (loads the reference read-only)

from hybfs import _native, csr, generator  # noqa: E402


def main():
    params = generator.GraphParams(scale=24, edgefactor=16, seed=1)
    rec = MG.big_config("S24", params, ["simd_a14b24"], roots_limit=4)
    e = generator.generate(params)
    g = csr.build(e)
    for s in rec["roots"]:
        par, _ = _native.bfs_reference(g.row_starts, g.adjacency, g.num_vertices, int(s))
        rec["roots"][s]["fifo_parent_sha"] = MG.sha(par)
    with open(os.path.join(HERE, "hashes_s24.json"), "w") as fh:
        json.dump({"S24_kron": rec}, fh, indent=1)
    print("wrote hashes_s24.json")


if __name__ == "__main__":
    main()
