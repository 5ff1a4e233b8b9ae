"""TEST/BASELINE INFRASTRUCTURE — the reference's CPU traversal, timed like the reference.

Drives the reference's own compiled layer kernels (``hybfs._native`` built from
/root/reference by oracle/build_ref.py) with a restatement of its Python
controller: hybrid.hybrid_bfs (hybrid.py:83-175), engine.run_* (engine.py:81-155),
engine._bu_aux (engine.py:29-57) and counters_after_layer (bfs_scalar.py:18-26,
including its O(n) Bitmap.indices() unpack, frontier.py:69-72, which is a large
part of the reference's cost).  Timing follows harness._run_one
(harness.py:224-244): perf_counter around the whole traversal, init included.

Used only by bench.py (``--impl reference`` and the cpu_baseline field) and
tests; never by the product.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import refnative

NIL = 0xFFFFFFFF


def _indices(words: np.ndarray, n: int) -> np.ndarray:
    flat = np.unpackbits(words.view(np.uint8), bitorder="little")
    return np.flatnonzero(flat[:n]).astype(np.uint32)


class RefGraph:
    """Reference-layout CSR plus the per-graph aux arrays of engine._bu_aux."""

    def __init__(self, row_starts: np.ndarray, adjacency: np.ndarray, m_edges: int):
        self.row_starts = np.ascontiguousarray(row_starts, dtype=np.int64)
        self.adjacency = np.ascontiguousarray(adjacency, dtype=np.uint32)
        self.n = len(self.row_starts) - 1
        self.m = int(m_edges)
        self._aux = {}

    def aux(self, max_pos: int):
        if max_pos in self._aux:
            return self._aux[max_pos]
        n = self.n
        nw = (n + 31) // 32
        rs32 = self.row_starts.astype(np.int32) if self.row_starts[n] <= 0x7FFFFFFF else None
        deg = np.diff(self.row_starts)

        def pack(flags):
            bits = np.zeros(nw * 32, dtype=bool)
            bits[:n] = flags
            return np.packbits(bits, bitorder="little").view(np.uint32)

        e = (rs32, pack(deg > 0), pack(deg > max_pos))
        self._aux[max_pos] = e
        return e


def hybrid_bfs(g: RefGraph, source: int, alpha: int = 1024, beta: int = 64,
               use_simd: bool = True, max_pos: int = 8):
    """One traversal with the reference rule (vertex counters); returns (parent, layers)."""
    nat = refnative.load()
    if nat is None:
        raise RuntimeError("reference _native not built (oracle/build_ref.py)")
    n = g.n
    rs, adj = g.row_starts, g.adjacency
    nw = (n + 31) // 32
    parent = np.full(n, NIL, dtype=np.uint32)
    parent[source] = source
    vis = np.zeros(nw, dtype=np.uint32)
    inw = np.zeros(nw, dtype=np.uint32)
    out = np.zeros(nw, dtype=np.uint32)
    vis[source >> 5] |= np.uint32(1 << (source & 31))
    inw[source >> 5] |= np.uint32(1 << (source & 31))
    e_u = n - 1
    v_f = 1
    bottom_up = False
    layers = 0
    while v_f > 0:
        f = e_u // alpha
        g_ = n // beta
        if v_f > f:
            bottom_up = True
        elif v_f < g_:
            bottom_up = False
        if bottom_up:
            if use_simd:
                rs32, posw, longw = g.aux(max_pos)
                nat.bottom_up_multiple_set(rs, adj, inw, vis, out, parent, n, max_pos, rs32, posw, longw)
            else:
                nat.bottom_up_layer(rs, adj, inw, vis, out, parent, n)
        else:
            if use_simd:
                nat.top_down_chunked(rs, adj, inw, vis, out, parent, n)
            else:
                nat.top_down_layer(rs, adj, inw, vis, out, parent, n)
        new = _indices(out, n).astype(np.int64)
        v_f = len(new)
        _e_f = int((rs[new + 1] - rs[new]).sum()) if v_f else 0
        e_u = n - int(np.bitwise_count(vis).sum())
        inw, out = out, inw
        out[:] = 0
        layers += 1
    return parent, layers


def time_roots(g: RefGraph, roots, alpha: int, beta: int, use_simd: bool = True):
    """Per-root wall seconds (harness._run_one timing), plus visited counts."""
    secs, reached = [], []
    for s in roots:
        t0 = time.perf_counter()
        parent, _ = hybrid_bfs(g, int(s), alpha=alpha, beta=beta, use_simd=use_simd)
        secs.append(time.perf_counter() - t0)
        reached.append(int(np.count_nonzero(parent != NIL)))
    return secs, reached


def cpu_info() -> dict:
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    nat = refnative.load()
    return {
        "cpu_model": model,
        "host_cores": os.cpu_count(),
        "variant": getattr(nat, "__variant__", None),
        "probe_uses_simd": bool(nat.probe_uses_simd()) if nat is not None else None,
    }
