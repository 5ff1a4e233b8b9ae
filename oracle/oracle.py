"""TEST INFRASTRUCTURE — ctypes wrapper over the C restatement ``hbfs_oracle.c``.

This is the CPU checker for the CUDA path (never the thing measured or shipped).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import it.  Each wrapper names the reference
function (file:line, relative to /root/reference/pkg/src/hybfs) it restates.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "hbfs_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

NIL = 0xFFFFFFFF
DEFAULT_PROBS = (0.57, 0.19, 0.19, 0.05)


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(
            ["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", SRC, "-o", LIB + ".tmp"],
            check=True,
        )
        os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB) and os.path.exists(SRC):
            build()
        L = C.CDLL(LIB)
        P = C.c_void_p
        i64, u64, i32 = C.c_int64, C.c_uint64, C.c_int
        L.hbo_mix64.restype = u64
        L.hbo_mix64.argtypes = [u64]
        L.hbo_generate.argtypes = [i32, i64, u64, P, i32, P, P]
        L.hbo_label_permutation.argtypes = [i64, u64, P]
        L.hbo_csr_build.restype = i64
        L.hbo_csr_build.argtypes = [P, P, i64, i64, i32, P, P]
        L.hbo_sample_sources.restype = i64
        L.hbo_sample_sources.argtypes = [P, i64, i64, u64, i32, P]
        L.hbo_bfs_reference.argtypes = [P, P, i64, i64, P, P]
        L.hbo_hybrid_bfs.restype = i64
        L.hbo_hybrid_bfs.argtypes = [P, P, i64, i64, i32, i32, i64, i64, i32, i32, i32, P, P, P, i64]
        L.hbo_minid_parents.argtypes = [P, P, i64, P, i64, P]
        L.hbo_td_layer.restype = i64
        L.hbo_td_layer.argtypes = [P, P, i64, P, P, P, P]
        L.hbo_bu_layer.argtypes = [P, P, i64, P, P, P, P]
        L.hbo_bu_multiple_set.argtypes = [P, P, i64, i32, P, P, P, P, P, P, P]
        L.hbo_validate_tree.restype = i32
        L.hbo_validate_tree.argtypes = [P, P, i64, i64, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


ROW_DTYPE = np.dtype(
    [
        ("layer", np.int32),
        ("direction", np.int32),
        ("v_f", np.int64),
        ("e_f", np.int64),
        ("e_u", np.int64),
        ("f_value", np.int64),
        ("g_value", np.int64),
        ("fallback_count", np.int64),
        ("gather_count", np.int64),
    ],
    align=True,
)


def mix64(x: int) -> int:
    return int(lib().hbo_mix64(x & 0xFFFFFFFFFFFFFFFF))


def thresholds(probs=DEFAULT_PROBS):
    """float64 {a, a+b, a+b+c} in Python's addition order (generator.py:149-150)."""
    a, b, c, _ = probs
    return np.array([a, a + b, a + b + c], dtype=np.float64)


def generate(scale: int, edgefactor: int = 16, seed: int = 1, probs=DEFAULT_PROBS,
             permute: bool = True):
    """generator.generate (generator.py:136-159) → (u, v) uint32 arrays."""
    m = (1 << scale) * edgefactor
    u = np.empty(m, dtype=np.uint32)
    v = np.empty(m, dtype=np.uint32)
    thr = thresholds(probs)
    lib().hbo_generate(scale, m, seed & 0xFFFFFFFFFFFFFFFF, _p(thr), int(permute), _p(u), _p(v))
    return u, v


def label_permutation(n: int, seed: int) -> np.ndarray:
    perm = np.empty(n, dtype=np.uint32)
    lib().hbo_label_permutation(n, seed & 0xFFFFFFFFFFFFFFFF, _p(perm))
    return perm


@dataclass
class HostCsr:
    num_vertices: int
    row_starts: np.ndarray  # int64[n+1]
    adjacency: np.ndarray  # uint32[arcs]
    in_edges_total: int

    @property
    def num_arcs(self) -> int:
        return int(self.row_starts[-1])

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_starts)


def csr_build(u, v, n: int, dedup: bool = False) -> HostCsr:
    """csr.from_arrays (csr.py:46-74); dedup = per-row unique + no self-loops."""
    u = np.ascontiguousarray(u, dtype=np.uint32)
    v = np.ascontiguousarray(v, dtype=np.uint32)
    m = len(u)
    rs = np.empty(n + 1, dtype=np.int64)
    adj = np.empty(max(2 * m, 1), dtype=np.uint32)
    arcs = lib().hbo_csr_build(_p(u), _p(v), m, n, int(dedup), _p(rs), _p(adj))
    return HostCsr(n, rs, adj[:arcs].copy() if arcs < len(adj) else adj, m)


def sample_sources(g: HostCsr, count: int, seed: int, allow_isolated: bool = False) -> np.ndarray:
    """harness.sample_sources (harness.py:73-97)."""
    out = np.empty(max(count, 1), dtype=np.uint32)
    k = lib().hbo_sample_sources(_p(g.row_starts), g.num_vertices, count,
                                 seed & 0xFFFFFFFFFFFFFFFF, int(allow_isolated), _p(out))
    if k < 0:
        raise ValueError("not enough eligible vertices")
    return out[:count]


def bfs_reference(g: HostCsr, source: int):
    """_native.bfs_reference (_native.pyx:39-62) → (parent, levels int32)."""
    n = g.num_vertices
    parent = np.empty(n, dtype=np.uint32)
    levels = np.empty(n, dtype=np.int32)
    lib().hbo_bfs_reference(_p(g.row_starts), _p(g.adjacency), n, source, _p(parent), _p(levels))
    return parent, levels


def hybrid_bfs(g: HostCsr, source: int, *, heuristic: str = "reference",
               counter_mode: str = "vertex", alpha: int = 1024, beta: int = 64,
               max_pos: int = 8, use_simd: bool = False, force_direction=None):
    """hybrid.hybrid_bfs (hybrid.py:83-175) → (parent, level, trace rows)."""
    n = g.num_vertices
    if not 0 <= source < n:
        raise IndexError(source)
    parent = np.empty(n, dtype=np.uint32)
    level = np.empty(n, dtype=np.int32)
    cap = 4096
    while True:
        rows = np.zeros(cap, dtype=ROW_DTYPE)
        fd = {None: -1, "top-down": 0, "bottom-up": 1}[force_direction]
        nl = lib().hbo_hybrid_bfs(
            _p(g.row_starts), _p(g.adjacency), n, source,
            1 if heuristic == "beamer" else 0, 1 if counter_mode == "edge" else 0,
            alpha, beta, max_pos, int(use_simd), fd, _p(parent), _p(level), _p(rows), cap,
        )
        if nl <= cap:
            return parent, level, rows[:nl]
        cap = int(nl)


def validate_tree(g: HostCsr, source: int, parent: np.ndarray):
    """harness.validate_tree (harness.py:129-205) → (rule or 0, witness)."""
    w = np.zeros(1, dtype=np.int64)
    parent = np.ascontiguousarray(parent, dtype=np.uint32)
    r = lib().hbo_validate_tree(_p(g.row_starts), _p(g.adjacency), g.num_vertices, source,
                                _p(parent), _p(w))
    return int(r), int(w[0])


def minid_parents(g: HostCsr, levels: np.ndarray, source: int) -> np.ndarray:
    """The F1 rule: parent[v] = min{u in Adj(v): level u = level v - 1}
    (the first such entry of the sorted row; C, OpenMP)."""
    n = g.num_vertices
    lv = np.ascontiguousarray(levels, dtype=np.int32)
    parent = np.empty(n, dtype=np.uint32)
    lib().hbo_minid_parents(_p(g.row_starts), _p(g.adjacency), n, _p(lv), int(source), _p(parent))
    return parent


# ---- per-layer steps (_native.pyx:65-239), in place on host arrays ----

def td_layer(rs, adj, n, inw, vis, out, parent) -> int:
    """top_down_layer / top_down_chunked (returns the chunked gather count)."""
    return int(lib().hbo_td_layer(_p(rs), _p(adj), n, _p(inw), _p(vis), _p(out), _p(parent)))


def bu_layer(rs, adj, n, inw, vis, out, parent) -> None:
    """bottom_up_layer."""
    lib().hbo_bu_layer(_p(rs), _p(adj), n, _p(inw), _p(vis), _p(out), _p(parent))


def bu_multiple_set(rs, adj, n, max_pos, posw, longw, inw, vis, out, parent):
    """bottom_up_multiple_set -> (fallback, gathers)."""
    fg = np.zeros(2, dtype=np.int64)
    lib().hbo_bu_multiple_set(_p(rs), _p(adj), n, max_pos, _p(posw), _p(longw), _p(inw), _p(vis),
                              _p(out), _p(parent), _p(fg))
    return int(fg[0]), int(fg[1])
