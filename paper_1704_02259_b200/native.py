"""The reference's compiled per-layer module ``hybfs._native`` (_native.pyx), on the GPU.

Same names, arguments, return values and in-place effects as the reference's
Cython kernels, so code (and tests) written against ``hybfs._native`` can call
these instead:

* ``bfs_reference(rs, adj, n, source) -> (parent, levels)`` (_native.pyx:39-62)
* ``top_down_layer(rs, adj, inw, visw, outw, parent, n) -> None`` (:65-86)
* ``bottom_up_layer(rs, adj, inw, visw, outw, parent, n) -> None`` (:89-104)
* ``bottom_up_multiple_set(rs, adj, inw, visw, outw, parent, n, max_pos,
  rs32_obj, posw, longw) -> (fallback, gathers)`` (:107-204)
* ``top_down_chunked(rs, adj, inw, visw, outw, parent, n) -> gathers`` (:207-239)
* ``probe_uses_simd() -> bool`` (:22-24)

Buffers are numpy arrays (copied to the device, results written back into the
caller's arrays) or CUDA tensors (updated in place on the device; uint32
buffers may be int32 tensors holding the same bits).  The dtype and layout
checks mirror the Cython buffer checks: a wrong dtype or a non-contiguous
buffer raises ``ValueError``.  All compute runs in libhbfs.so
(csrc/layer.cu); there is no CPU path.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

__all__ = [
    "bfs_reference", "bottom_up_layer", "bottom_up_multiple_set", "probe_uses_simd",
    "top_down_chunked", "top_down_layer",
]


def probe_uses_simd() -> bool:
    """The bottom-up probe is a vectorised (warp-wide) gather on the GPU."""
    return True


def _torch():
    import torch

    return torch


def _is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


_NP = {"i64": np.int64, "u32": np.uint32, "i32": np.int32}


def _dev(x, kind: str, name: str, writable: bool):
    """(device tensor, numpy array to write back or None)."""
    torch = _torch()
    if _is_tensor(x):
        ok = {"i64": (torch.int64,), "u32": (torch.int32, getattr(torch, "uint32", torch.int32)),
              "i32": (torch.int32,)}[kind]
        if x.dtype not in ok:
            raise ValueError(f"Buffer dtype mismatch for {name}: {x.dtype}")
        if not x.is_cuda:
            raise ValueError(f"{name}: CPU tensors are not accepted (pass numpy or a CUDA tensor)")
        if not x.is_contiguous():
            raise ValueError(f"{name}: buffer is not C-contiguous")
        return x, None
    a = np.asarray(x)
    if a.dtype != _NP[kind]:
        raise ValueError(f"Buffer dtype mismatch for {name}: expected {np.dtype(_NP[kind])}, got {a.dtype}")
    if a.ndim != 1 or not a.flags.c_contiguous:
        raise ValueError(f"{name}: buffer is not a C-contiguous 1-d array")
    if writable and not a.flags.writeable:
        raise ValueError(f"{name}: buffer is read-only")
    view = a.view(np.int32) if kind == "u32" else a
    t = torch.from_numpy(view.copy()).cuda() if a.size else torch.empty(1, dtype=torch.int32 if kind != "i64" else torch.int64, device="cuda")
    return t, (a if writable else None)


def _back(t, host):
    if host is not None and host.size:
        out = t[: host.size].cpu().numpy()
        host[...] = out.view(host.dtype)


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def _size(x) -> int:
    return int(x.numel()) if _is_tensor(x) else int(np.asarray(x).size)


def _check_sizes(rs, inw, visw, outw, parent, n: int, adj=None) -> None:
    """The Cython kernels trust their buffers; the device kernels must not
    read or write past them, so the lengths the loops touch are checked."""
    n = int(n)
    if n < 0:
        raise ValueError("n must be >= 0")
    nw = (n + 31) // 32
    if _size(rs) < n + 1:
        raise ValueError(f"rs has {_size(rs)} entries, needs n + 1 = {n + 1}")
    for name, x in (("inw", inw), ("visw", visw), ("outw", outw)):
        if _size(x) < nw:
            raise ValueError(f"{name} has {_size(x)} words, needs ceil(n/32) = {nw}")
    if _size(parent) < n:
        raise ValueError(f"parent has {_size(parent)} entries, needs n = {n}")
    if adj is not None and n > 0:
        arcs = int(rs[n].item()) if _is_tensor(rs) else int(np.asarray(rs)[n])
        if _size(adj) < arcs:
            raise ValueError(f"adj has {_size(adj)} entries, rs[n] = {arcs}")


def _layer_buffers(rs, adj, inw, visw, outw, parent, n):
    _check_sizes(rs, inw, visw, outw, parent, n, adj)
    lib = _lib.load(require_device=True)
    bufs = [_dev(rs, "i64", "rs", False), _dev(adj, "u32", "adj", False), _dev(inw, "u32", "inw", False),
            _dev(visw, "u32", "visw", True), _dev(outw, "u32", "outw", True),
            _dev(parent, "u32", "parent", True)]
    return lib, bufs


def _finish(bufs):
    for t, host in bufs[3:]:
        _back(t, host)


def top_down_layer(rs, adj, inw, visw, outw, parent, n: int) -> None:
    """Scalar top-down layer over bitmap frontiers (_native.pyx:65-86)."""
    top_down_chunked(rs, adj, inw, visw, outw, parent, n)


def top_down_chunked(rs, adj, inw, visw, outw, parent, n: int) -> int:
    """Chunked top-down layer; returns gather_count (_native.pyx:207-239)."""
    lib, b = _layer_buffers(rs, adj, inw, visw, outw, parent, n)
    g = C.c_int64()
    _lib.check(lib.hbfs_layer_top_down(*(_ptr(t) for t, _ in b), int(n), C.byref(g),
                                       _lib.current_stream()))
    _finish(b)
    return g.value


def bottom_up_layer(rs, adj, inw, visw, outw, parent, n: int) -> None:
    """Scalar bottom-up layer: masked full scan of all vertices (_native.pyx:89-104)."""
    lib, b = _layer_buffers(rs, adj, inw, visw, outw, parent, n)
    _lib.check(lib.hbfs_layer_bottom_up(*(_ptr(t) for t, _ in b), int(n), 1, None, None,
                                        _lib.current_stream()))
    _finish(b)


def bottom_up_multiple_set(rs, adj, inw, visw, outw, parent, n: int, max_pos: int, rs32_obj, posw,
                           longw) -> tuple[int, int]:
    """16-lane bottom-up layer; returns (fallback_count, gather_count)
    (_native.pyx:107-204).  rs32_obj/posw/longw only select and prune work in
    the reference; the GPU derives the same from the row starts."""
    if int(max_pos) < 1:
        raise ValueError("max_pos must be >= 1")
    for name, x in (("posw", posw), ("longw", longw)):
        if _is_tensor(x):
            _dev(x, "u32", name, False)
        elif np.asarray(x).dtype != np.uint32:
            raise ValueError(f"Buffer dtype mismatch for {name}")
    if rs32_obj is not None and not _is_tensor(rs32_obj) and np.asarray(rs32_obj).dtype != np.int32:
        raise ValueError("Buffer dtype mismatch for rs32_obj")
    if _is_tensor(adj):
        if adj.numel() == 0:
            return 0, 0
    elif np.asarray(adj).size == 0:
        return 0, 0
    lib, b = _layer_buffers(rs, adj, inw, visw, outw, parent, n)
    fb, ga = C.c_int64(), C.c_int64()
    _lib.check(lib.hbfs_layer_bottom_up(*(_ptr(t) for t, _ in b), int(n), int(max_pos), C.byref(fb),
                                        C.byref(ga), _lib.current_stream()))
    _finish(b)
    return fb.value, ga.value


def bfs_reference(rs, adj, n: int, source: int):
    """Sequential queue-based BFS; returns (parent uint32[n], levels int32[n])
    (_native.pyx:39-62): levels, and the FIFO queue's first-discoverer parents."""
    n = int(n)
    if n <= 0 or _size(rs) < n + 1:
        raise ValueError("rs must hold n + 1 >= 2 row starts")
    arcs = int(rs[n].item()) if _is_tensor(rs) else int(np.asarray(rs)[n])
    if _size(adj) < arcs:
        raise ValueError(f"adj has {_size(adj)} entries, rs[n] = {arcs}")
    lib = _lib.load(require_device=True)
    torch = _torch()
    trs, _ = _dev(rs, "i64", "rs", False)
    tadj, _ = _dev(adj, "u32", "adj", False)
    n = int(n)
    par = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    lev = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    _lib.check(lib.hbfs_reference_bfs(_ptr(trs), _ptr(tadj), n, int(source), _ptr(par), _ptr(lev),
                                      _lib.current_stream()))
    return par[:n].cpu().numpy().view(np.uint32), lev[:n].cpu().numpy()
