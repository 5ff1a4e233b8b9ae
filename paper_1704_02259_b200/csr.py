"""Device-resident CSR graph — the reference's ``hybfs.csr`` API (csr.py:18-78)
backed by libhbfs.

``build`` / ``from_arrays`` construct the CSR on the GPU (radix sort of both
arc directions, csrc/graph.cu) bit-exactly like ``csr.from_arrays``
(csr.py:46-74): duplicates and self-loops kept, rows ascending.  ``dedup=True``
gives the BASELINE.json variant (per-row unique, self-loops dropped).
``generate_graph`` runs generator + build without leaving the device.
``from_csr`` imports any reference-layout CSR (e.g. a ``hybfs.CsrGraph``).
Host copies of ``row_starts`` / ``adjacency`` are exported lazily.
"""

from __future__ import annotations

import ctypes as C
import struct
import weakref

import numpy as np

from . import _lib
from .generator import CapacityError, EdgeList, GraphParams, thresholds


class CsrGraph:
    """CSR over ``num_vertices`` vertices living on the current CUDA device."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        lib = _lib.load()
        n, arcs, m, md = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        wide = C.c_int32()
        _lib.check(lib.hbfs_graph_info(handle, C.byref(n), C.byref(arcs), C.byref(m),
                                       C.byref(md), C.byref(wide)))
        self.num_vertices = int(n.value)
        self.num_arcs = int(arcs.value)
        self.in_edges_total = int(m.value)
        self.max_degree = int(md.value)
        self.wide_offsets = bool(wide.value)
        self._rs = None
        self._adj = None

    # -- lifetime
    @property
    def handle(self) -> C.c_void_p:
        if self._h is None:
            raise RuntimeError("graph has been freed")
        return self._h

    def free(self) -> None:
        if self._h is not None:
            _lib.load().hbfs_graph_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    # -- reference accessors (csr.py:25-38)
    @property
    def row_starts(self) -> np.ndarray:
        if self._rs is None:
            self._export()
        return self._rs

    @property
    def adjacency(self) -> np.ndarray:
        if self._adj is None:
            self._export()
        return self._adj

    def _export(self) -> None:
        rs = np.empty(self.num_vertices + 1, dtype=np.int64)
        adj = np.empty(self.num_arcs, dtype=np.uint32)
        _lib.check(_lib.load().hbfs_graph_export(self.handle, rs.ctypes.data_as(C.c_void_p),
                                                 adj.ctypes.data_as(C.c_void_p), 0, None))
        rs.setflags(write=False)
        adj.setflags(write=False)
        self._rs, self._adj = rs, adj

    def degree(self, v: int) -> int:
        if not 0 <= v < self.num_vertices:
            raise IndexError(f"vertex {v} out of range [0, {self.num_vertices})")
        return int(self.row_starts[v + 1] - self.row_starts[v])

    def row(self, v: int) -> np.ndarray:
        if not 0 <= v < self.num_vertices:
            raise IndexError(f"vertex {v} out of range [0, {self.num_vertices})")
        return self.adjacency[self.row_starts[v]: self.row_starts[v + 1]]

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_starts)

    def __repr__(self) -> str:
        return (f"CsrGraph(n={self.num_vertices}, arcs={self.num_arcs}, "
                f"m={self.in_edges_total}, device)")


def _new(fn, *args) -> CsrGraph:
    h = C.c_void_p()
    _lib.check(fn(*args, C.byref(h)))
    return CsrGraph(h)


def from_arrays(eu, ev, n: int, dedup: bool = False) -> CsrGraph:
    """CSR from endpoint arrays (csr.py:46-74), built on the device."""
    lib = _lib.load(require_device=True)
    if n > 1 << 32:
        raise CapacityError("vertex ids are 32-bit; at most 2^32 vertices")
    eu = np.ascontiguousarray(eu, dtype=np.uint32)
    ev = np.ascontiguousarray(ev, dtype=np.uint32)
    if len(eu) != len(ev):
        raise ValueError("endpoint arrays differ in length")
    if len(eu) and (int(eu.max()) >= n or int(ev.max()) >= n):
        raise ValueError("endpoint id out of range")
    return _new(lib.hbfs_graph_build, eu.ctypes.data_as(C.c_void_p), ev.ctypes.data_as(C.c_void_p),
                len(eu), n, int(dedup), 0, None)


def build(edges: EdgeList, dedup: bool = False) -> CsrGraph:
    """CSR from an EdgeList (csr.py:41-43)."""
    return from_arrays(edges.u, edges.v, edges.num_vertices, dedup=dedup)


def generate_graph(params: GraphParams, dedup: bool = False) -> CsrGraph:
    """generate + build entirely on the device (no host edge list)."""
    lib = _lib.load(require_device=True)
    if params.scale > 32:
        raise CapacityError("vertex ids are 32-bit")
    thr = thresholds(params.probs)
    return _new(lib.hbfs_graph_generate, params.scale, params.edgefactor,
                params.seed & 0xFFFFFFFFFFFFFFFF, thr.ctypes.data_as(C.c_void_p),
                int(params.permute_labels), int(dedup), None)


def from_csr(row_starts, adjacency, in_edges_total: int | None = None) -> CsrGraph:
    """Import a reference-layout CSR (int64 row_starts, uint32 adjacency)."""
    lib = _lib.load(require_device=True)
    rs = np.ascontiguousarray(row_starts, dtype=np.int64)
    adj = np.ascontiguousarray(adjacency, dtype=np.uint32)
    n = len(rs) - 1
    if n < 0 or int(rs[-1]) != len(adj):
        raise ValueError("row_starts[-1] must equal len(adjacency)")
    m = len(adj) // 2 if in_edges_total is None else int(in_edges_total)
    return _new(lib.hbfs_graph_from_csr, rs.ctypes.data_as(C.c_void_p),
                adj.ctypes.data_as(C.c_void_p), n, m, 0, None)


def as_device_graph(g) -> CsrGraph:
    """Accept our CsrGraph or any object with the reference CsrGraph fields."""
    if isinstance(g, CsrGraph):
        return g
    key = id(g)
    cache = _IMPORTED.get(key)
    if cache is not None and cache[0]() is g:
        return cache[1]
    dg = from_csr(g.row_starts, g.adjacency, getattr(g, "in_edges_total", None))
    try:
        ref = weakref.ref(g)
        # the device copy (and its workspace) is freed with the host graph
        weakref.finalize(g, _drop_imported, key, dg)
    except TypeError:  # not weak-referenceable: keep only the latest import
        for k in [k for k, v in _IMPORTED.items() if v[2]]:
            _drop_imported(k, _IMPORTED[k][1])
        ref = (lambda obj: (lambda: obj))(g)
        _IMPORTED[key] = (ref, dg, True)
        return dg
    _IMPORTED[key] = (ref, dg, False)
    return dg


# id(host graph) -> (weak reference, device CsrGraph, strongly held?)
_IMPORTED: dict = {}


def _drop_imported(key, dg) -> None:
    cur = _IMPORTED.get(key)
    if cur is not None and cur[1] is dg:
        del _IMPORTED[key]
    dg.free()


def degree(g: CsrGraph, v: int) -> int:
    return g.degree(v)


# ---------------------------------------------------------------- CSR cache
# a CSR blob next to the reference's HBFSEDG1 edge-list dump
# (generator.py:162-187), so large graphs are built once.  Layout (little
# endian): magic "HBFSCSR1", header <QQQIIQ8d> = n, arcs, m_edges, scale,
# flags (bit0 dedup, bit1 permute_labels), seed, edgefactor, probs[4] and 3
# reserved doubles; then int64 row_starts[n+1], uint32 adjacency[arcs].

_CSR_MAGIC = b"HBFSCSR1"
_CSR_HEADER = struct.Struct("<8sQQQIIQd4d3d")


def save(g, path, params: GraphParams | None = None, dedup: bool = False) -> None:
    """Write the CSR of `g` (our CsrGraph or any object with the reference
    CsrGraph fields) to `path`."""
    rs = np.ascontiguousarray(g.row_starts, dtype=np.int64)
    adj = np.ascontiguousarray(g.adjacency, dtype=np.uint32)
    n = len(rs) - 1
    m = int(getattr(g, "in_edges_total", len(adj) // 2))
    probs = tuple(params.probs) if params else (0.0, 0.0, 0.0, 0.0)
    flags = (1 if dedup else 0) | (2 if (params is None or params.permute_labels) else 0)
    with open(path, "wb") as fh:
        fh.write(_CSR_HEADER.pack(_CSR_MAGIC, n, len(adj), m, params.scale if params else 0, flags,
                                  params.seed if params else 0,
                                  float(params.edgefactor) if params else 0.0, *probs, 0.0, 0.0, 0.0))
        rs.tofile(fh)
        adj.tofile(fh)


def load_arrays(path):
    """Read a CSR blob -> (row_starts, adjacency, m_edges, meta dict)."""
    with open(path, "rb") as fh:
        hdr = _CSR_HEADER.unpack(fh.read(_CSR_HEADER.size))
        if hdr[0] != _CSR_MAGIC:
            raise ValueError(f"bad magic {hdr[0]!r}")
        n, arcs, m, scale, flags, seed, ef = hdr[1:8]
        probs = tuple(hdr[8:12])
        rs = np.fromfile(fh, dtype="<i8", count=n + 1)
        adj = np.fromfile(fh, dtype="<u4", count=arcs)
    if len(rs) != n + 1 or len(adj) != arcs or int(rs[-1]) != arcs:
        raise ValueError("truncated or inconsistent CSR blob")
    meta = dict(scale=scale, dedup=bool(flags & 1), permute_labels=bool(flags & 2), seed=seed,
                edgefactor=int(ef), probs=probs)
    return rs, adj, int(m), meta


def load(path) -> CsrGraph:
    """CSR blob -> device graph."""
    rs, adj, m, _ = load_arrays(path)
    return from_csr(rs, adj, m)
