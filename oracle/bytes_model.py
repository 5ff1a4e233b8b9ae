"""TEST INFRASTRUCTURE — numpy restatement of the algorithmic byte model
(SURVEY §8(d)): B_sector (unique 32-byte sectors touched) and B_useful (bytes
without sector rounding) of one traversal, from the graph, the level array and
the per-layer directions.  Checks csrc/validate.cu `hbfs_traversal_bytes`, the
numerator of bench.py's roofline.  Small graphs only (vectorised but O(arcs)
memory per layer)."""

from __future__ import annotations

import numpy as np


def _sec(b: int) -> int:
    return (b + 31) // 32 * 32


def _rows(rs: np.ndarray, verts: np.ndarray, lens: np.ndarray) -> np.ndarray:
    """Arc positions rs[v] .. rs[v] + lens[v] - 1 for every v, concatenated."""
    lens = lens.astype(np.int64)
    if lens.sum() == 0:
        return np.zeros(0, dtype=np.int64)
    starts = rs[verts].astype(np.int64)
    off = np.repeat(starts - np.concatenate(([0], np.cumsum(lens)[:-1])), lens)
    return np.arange(int(lens.sum()), dtype=np.int64) + off


def traversal_bytes(rs, adj, level, directions, rs_bytes: int = 4) -> tuple[int, int]:
    """directions: per layer, 0 = top-down, 1 = bottom-up (layer L expands depth L)."""
    rs = np.asarray(rs, dtype=np.int64)
    adj = np.asarray(adj, dtype=np.int64)
    level = np.asarray(level, dtype=np.int64)
    n = len(rs) - 1
    W = (n + 31) // 32
    deg = np.diff(rs)
    bs = bu = 8 * n + 12 * W  # B_init: parent + level + three bitmaps
    for L, d in enumerate(directions):
        newv = np.flatnonzero(level == L + 1)
        N = len(newv)
        s_pl = 2 * 32 * len(np.unique(newv * 4 // 32))  # parent[N] and level[N]
        if d == 0:  # top-down: frontier F = depth L
            F = np.flatnonzero(level == L)
            mf = int(deg[F].sum())
            rs_sec = np.unique(np.concatenate((F * rs_bytes // 32, (F + 1) * rs_bytes // 32)))
            k = _rows(rs, F, deg[F])
            adj_sec = np.unique(k * 4 // 32)
            bm_sec = np.unique((adj[k] >> 5) * 4 // 32)
            bs += _sec(4 * len(F)) + 32 * (len(rs_sec) + len(adj_sec) + len(bm_sec)) + s_pl + _sec(4 * N)
            bu += 20 * len(F) + 4 * mf + 12 * N
        else:  # bottom-up: U = unvisited before the layer
            Umask = (level == -1) | (level > L)
            U = int(Umask.sum())
            V = np.flatnonzero(Umask & (deg > 0))
            rs_sec = np.unique(np.concatenate((V * rs_bytes // 32, (V + 1) * rs_bytes // 32)))
            probes = deg[V].copy()
            found = level[V] == L + 1
            for i in np.flatnonzero(found):  # 1 + first depth-L entry of the sorted row
                v = V[i]
                row = adj[rs[v]:rs[v + 1]]
                probes[i] = int(np.flatnonzero(level[row] == L)[0]) + 1
            k = _rows(rs, V, probes)
            adj_sec = np.unique(k * 4 // 32)
            bm_sec = np.unique((adj[k] >> 5) * 4 // 32)
            bs += 4 * W + 32 * (len(rs_sec) + len(adj_sec) + len(bm_sec)) + s_pl + 4 * W
            bu += 8 * W + 8 * U + 4 * int(probes.sum()) + 8 * N
    return int(bs), int(bu)
