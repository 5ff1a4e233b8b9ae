"""Golden per-layer vectors from the REFERENCE's compiled kernels (build container only).

Runs the reference's own ``hybfs._native`` (compiled from /root/reference by
oracle/build_ref.py, loaded by oracle/refnative.py) on small graphs generated
by the oracle (bit-exact with the reference generator, pinned by small.npz) and
records into ``layers.npz``:

* ``bfs_reference`` parents (FIFO first-discoverer rule) and levels;
* for every layer d of a traversal: the inputs (frontier = level d, visited =
  level <= d, out = a few junk bits, parent = seeded junk) and the in-place
  results of ``top_down_layer``, ``top_down_chunked`` (+ gathers),
  ``bottom_up_layer`` and ``bottom_up_multiple_set`` (+ fallback, gathers) at
  several max_pos values.

Usage: python tests/golden/make_layers_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import oracle as O  # noqa: E402
from oracle import refnative  # noqa: E402

GRAPHS = [
    # name, scale, edgefactor, seed, probs
    ("k8", 8, 8, 5, (0.57, 0.19, 0.19, 0.05)),
    ("u9", 9, 4, 3, (0.25, 0.25, 0.25, 0.25)),
    ("k10", 10, 16, 1, (0.57, 0.19, 0.19, 0.05)),
]
MAX_POS = (1, 3, 8, 16)


def bits_of(mask: np.ndarray, nw: int) -> np.ndarray:
    w = np.zeros(nw * 32, dtype=np.uint8)
    w[: len(mask)] = mask
    return np.packbits(w, bitorder="little").view(np.uint32).copy()


def main():
    nat = refnative.load()
    assert nat is not None, "build the reference kernels first (oracle/build_ref.py)"
    out = {}
    rng = np.random.default_rng(1704)
    for name, scale, ef, seed, probs in GRAPHS:
        u, v = O.generate(scale, ef, seed, probs)
        n = 1 << scale
        g = O.csr_build(u, v, n)
        rs, adj = g.row_starts, g.adjacency
        nw = (n + 31) // 32
        out[f"{name}/rs"] = rs
        out[f"{name}/adj"] = adj
        deg = np.diff(rs)
        posw = bits_of(deg > 0, nw)
        srcs = O.sample_sources(g, 2, seed)
        out[f"{name}/sources"] = srcs
        for s in srcs:
            s = int(s)
            par, lev = nat.bfs_reference(rs, adj, n, s)
            out[f"{name}/{s}/ref_parent"] = par
            out[f"{name}/{s}/ref_level"] = lev
            for d in range(int(lev.max()) + 1):
                key = f"{name}/{s}/{d}"
                inw = bits_of(lev == d, nw)
                vis0 = bits_of((lev >= 0) & (lev <= d), nw)
                out0 = np.zeros(nw, dtype=np.uint32)
                out0[rng.integers(0, nw, 2)] |= rng.integers(1, 1 << 31, 2).astype(np.uint32)
                out0 &= ~vis0  # junk on unvisited, undiscovered bits only where harmless
                par0 = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
                out[key + "/in"] = inw
                out[key + "/vis"] = vis0
                out[key + "/out"] = out0
                out[key + "/parent"] = par0
                for kern in ("td", "tdc", "bu"):
                    vi, ou, pa = vis0.copy(), out0.copy(), par0.copy()
                    if kern == "td":
                        nat.top_down_layer(rs, adj, inw, vi, ou, pa, n)
                    elif kern == "tdc":
                        out[key + "/tdc/gathers"] = np.int64(nat.top_down_chunked(rs, adj, inw, vi, ou, pa, n))
                    else:
                        nat.bottom_up_layer(rs, adj, inw, vi, ou, pa, n)
                    out[f"{key}/{kern}/vis"], out[f"{key}/{kern}/out"], out[f"{key}/{kern}/parent"] = vi, ou, pa
                for mp in MAX_POS:
                    vi, ou, pa = vis0.copy(), out0.copy(), par0.copy()
                    longw = bits_of(deg > mp, nw)
                    rs32 = rs.astype(np.int32)
                    fb, ga = nat.bottom_up_multiple_set(rs, adj, inw, vi, ou, pa, n, mp, rs32, posw, longw)
                    k2 = f"{key}/bums{mp}"
                    out[k2 + "/vis"], out[k2 + "/out"], out[k2 + "/parent"] = vi, ou, pa
                    out[k2 + "/counters"] = np.array([fb, ga], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "layers.npz"), **out)
    print(f"wrote layers.npz: {len(out)} arrays")


if __name__ == "__main__":
    main()
