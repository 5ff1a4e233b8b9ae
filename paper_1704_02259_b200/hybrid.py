"""Hybrid BFS controller API — ``hybfs.hybrid`` (hybrid.py:27-175) on the GPU.

``hybrid_bfs`` keeps the reference's signature and return value
``(BfsTree, [LayerTraceRow])``; the traversal, the per-layer counters and the
direction decision all run inside one persistent CUDA kernel (csrc/bfs.cu),
so the host sees no per-layer round trip.  ``bfs`` is the new entry point the
north star asks for: parent and level arrays (device tensors by default).

Heuristics:
* ``"reference"`` — the reference's rule (hybrid.py:72-80): BU if
  n_f > e_u // alpha, TD if n_f < n // beta, else keep; e_u per counter_mode.
* ``"beamer"`` — Beamer's rule with the GAP guard: TD->BU when
  m_f > m_u // alpha; BU->TD when the frontier shrinks and n_f <= n // beta;
  m_u is the edge-denominated unvisited count.
Parents are identical in every mode (min-id rule) with
``parent_mode="minid"``; ``"any"`` lets the first claimer win.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib, engine
from .csr import as_device_graph
from .frontier import BfsTree, LayerCounters
from .lanes import VecConfig

TOP_DOWN = "top-down"
BOTTOM_UP = "bottom-up"
COUNTER_MODES = ("vertex", "edge")
HEURISTICS = ("reference", "beamer")
PARENT_MODES = ("minid", "any")


@dataclass
class HeuristicParams:
    """Switching thresholds (hybrid.py:27-44) plus the heuristic family."""

    alpha: int = 1024
    beta: int = 64
    counter_mode: str = "vertex"
    heuristic: str = "reference"

    def __post_init__(self):
        if self.alpha < 1 or self.beta < 1:
            raise ValueError("alpha and beta must be >= 1")
        if self.counter_mode not in COUNTER_MODES:
            raise ValueError(f"counter_mode must be one of {COUNTER_MODES}")
        if self.heuristic not in HEURISTICS:
            raise ValueError(f"heuristic must be one of {HEURISTICS}")


@dataclass
class LayerTraceRow:
    layer: int
    direction: str
    kernel: str  # "scalar" | "simd"
    v_f: int
    e_f: int
    e_u: int
    f_value: int
    g_value: int
    elapsed: float
    fallback_count: int = 0
    gather_count: int = 0


def f_threshold(p: HeuristicParams, n: int, c: LayerCounters) -> int:
    return c.e_u // p.alpha


def g_threshold(p: HeuristicParams, n: int, c: LayerCounters) -> int:
    return n // p.beta


def decide(p: HeuristicParams, current: str, frontier_size: int, n: int, c: LayerCounters) -> str:
    """Host restatement of the reference rule (hybrid.py:72-80); the device
    evaluates the same rule (csrc/bfs.cu ``decide``)."""
    if frontier_size > f_threshold(p, n, c):
        return BOTTOM_UP
    if frontier_size < g_threshold(p, n, c):
        return TOP_DOWN
    return current


def _params(p: HeuristicParams, cfg: VecConfig, use_simd: bool, force_direction,
            parent_mode: str) -> _lib.hbfs_params:
    if force_direction not in (None, TOP_DOWN, BOTTOM_UP):
        raise ValueError(f"force_direction must be None, {TOP_DOWN!r} or {BOTTOM_UP!r}")
    if parent_mode not in PARENT_MODES:
        raise ValueError(f"parent_mode must be one of {PARENT_MODES}")
    hp = _lib.hbfs_params()
    hp.heuristic = HEURISTICS.index(p.heuristic)
    hp.counter_mode = COUNTER_MODES.index(p.counter_mode)
    hp.alpha = p.alpha
    hp.beta = p.beta
    hp.max_pos = cfg.max_pos
    hp.use_simd = int(bool(use_simd))
    hp.force_direction = {None: -1, TOP_DOWN: 0, BOTTOM_UP: 1}[force_direction]
    hp.parent_mode = PARENT_MODES.index(parent_mode)
    return hp


@dataclass
class BfsResult:
    parent: object  # torch.int32 tensor (bit pattern of uint32) or numpy uint32
    level: object   # torch.int32 tensor or numpy int32
    trace: list
    device_seconds: float


_TRACE_CAP = 4096
_tls = threading.local()
_PINNED_MIN_N = 1 << 16


def _host_parent(n: int) -> np.ndarray:
    """Result array for hybrid_bfs.  Large outputs come from torch's caching
    pinned-host allocator, so the device-to-host copy runs at full PCIe rate
    (pageable memory takes a driver staging copy); the block returns to the
    cache when the caller drops the array (the ndarray holds the tensor).
    Cached pinned blocks stay page-locked until the process exits; callers that
    keep many trees alive can set HBFS_PINNED_RESULTS=0 for pageable arrays."""
    if n >= _PINNED_MIN_N and os.environ.get("HBFS_PINNED_RESULTS", "1") != "0":
        import torch

        return torch.empty(n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    return np.empty(n, dtype=np.uint32)


def _run(g, source: int, hp: _lib.hbfs_params, parent, level, on_device: bool, want_trace: bool,
         use_simd: bool):
    lib = _lib.load(require_device=True)
    n_layers = C.c_int64()
    ms = C.c_float()
    cap = _TRACE_CAP if want_trace else 0
    rows = getattr(_tls, "rows", None)  # reused per thread: rows are copied out below
    if rows is None:
        rows = _tls.rows = (_lib.hbfs_layer_row * _TRACE_CAP)()
    pp = C.c_void_p(parent) if isinstance(parent, int) else parent
    lp = C.c_void_p(level) if isinstance(level, int) else level
    stream = _lib.current_stream() if on_device else None
    _lib.check(lib.hbfs_bfs(g.handle, source, C.byref(hp), pp, lp, int(on_device),
                            rows if want_trace else None, cap, C.byref(n_layers), C.byref(ms),
                            stream))
    if want_trace and n_layers.value > cap:
        # pathological depth (> trace cap): rerun with a trace buffer that fits
        cap = int(n_layers.value)
        rows = (_lib.hbfs_layer_row * cap)()
        _lib.check(lib.hbfs_bfs(g.handle, source, C.byref(hp), pp, lp, int(on_device), rows, cap,
                                C.byref(n_layers), C.byref(ms), stream))
    trace = []
    if want_trace:
        kern = "simd" if use_simd else "scalar"
        for i in range(n_layers.value):
            r = rows[i]
            trace.append(LayerTraceRow(
                layer=r.layer, direction=BOTTOM_UP if r.direction else TOP_DOWN, kernel=kern,
                v_f=r.v_f, e_f=r.e_f, e_u=r.e_u, f_value=r.f_value, g_value=r.g_value,
                elapsed=r.elapsed, fallback_count=r.fallback_count, gather_count=r.gather_count))
    return trace, ms.value * 1e-3


def hybrid_bfs(g, source: int, p: HeuristicParams | None = None, cfg: VecConfig | None = None,
               use_simd: bool = False, engine_name: str = "auto",
               force_direction: str | None = None, parent_mode: str = "minid", out=None):
    """Full traversal (hybrid.py:83-175) → (BfsTree, trace).

    Parents only, as the reference's ``BfsTree`` (frontier.py:95-107); no level
    array is produced.  ``out`` reuses a host uint32[n] buffer (e.g. pinned)."""
    p = p if p is not None else HeuristicParams()
    cfg = cfg if cfg is not None else VecConfig()
    engine.resolve_engine(engine_name, cfg.backend)
    dg = as_device_graph(g)
    n = dg.num_vertices
    if not 0 <= source < n:
        raise IndexError(f"source {source} out of range [0, {n})")
    hp = _params(p, cfg, use_simd, force_direction, parent_mode)
    if out is None:
        parent = _host_parent(n)
    else:
        parent = out
        if parent.dtype != np.uint32 or parent.shape != (n,) or not parent.flags.c_contiguous:
            raise ValueError("out must be a contiguous uint32 array of length n")
    trace, _ = _run(dg, int(source), hp, parent.ctypes.data_as(C.c_void_p), None, False, True,
                    use_simd)
    return BfsTree(parent=parent, source=int(source)), trace


def _check_device_out(t, name: str, n: int, dtypes) -> None:
    """A device output buffer: CUDA tensor on the current device, shape (n,),
    4-byte integer dtype, contiguous (the kernel writes n entries)."""
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"out {name}: expected a CUDA tensor")
    if t.device.index != torch.cuda.current_device():
        raise ValueError(f"out {name}: tensor is on {t.device}, not the current device")
    if t.dtype not in dtypes or tuple(t.shape) != (n,) or not t.is_contiguous():
        raise ValueError(f"out {name}: expected a contiguous {dtypes[0]} tensor of shape ({n},)")


def _check_host_out(a, name: str, n: int, dtype) -> None:
    if not isinstance(a, np.ndarray) or a.dtype != dtype or a.shape != (n,) or \
            not a.flags.c_contiguous or not a.flags.writeable:
        raise ValueError(f"out {name}: expected a writable contiguous {np.dtype(dtype)} array of length {n}")


def bfs(g, root: int, p: HeuristicParams | None = None, cfg: VecConfig | None = None,
        use_simd: bool = True, force_direction: str | None = None, parent_mode: str = "minid",
        device: bool = True, trace: bool = True, out=None) -> BfsResult:
    """bfs(root) → parent (uint32 bits) and level (int32) arrays.

    device=True returns torch CUDA tensors (int32; view parent bits as uint32);
    device=False returns numpy arrays.  ``out=(parent, level)`` reuses buffers.
    """
    p = p if p is not None else HeuristicParams()
    cfg = cfg if cfg is not None else VecConfig()
    dg = as_device_graph(g)
    n = dg.num_vertices
    if not 0 <= root < n:
        raise IndexError(f"source {root} out of range [0, {n})")
    hp = _params(p, cfg, use_simd, force_direction, parent_mode)
    if device:
        import torch

        if out is not None:
            parent, level = out
            _check_device_out(parent, "parent", n, (torch.int32, getattr(torch, "uint32", torch.int32)))
            _check_device_out(level, "level", n, (torch.int32,))
        else:
            parent = torch.empty(n, dtype=torch.int32, device="cuda")
            level = torch.empty(n, dtype=torch.int32, device="cuda")
        tr, secs = _run(dg, int(root), hp, parent.data_ptr(), level.data_ptr(), True, trace,
                        use_simd)
    else:
        if out is not None:
            parent, level = out
            _check_host_out(parent, "parent", n, np.uint32)
            _check_host_out(level, "level", n, np.int32)
        else:
            parent = np.empty(n, dtype=np.uint32)
            level = np.empty(n, dtype=np.int32)
        tr, secs = _run(dg, int(root), hp, parent.ctypes.data_as(C.c_void_p),
                        level.ctypes.data_as(C.c_void_p), False, trace, use_simd)
    return BfsResult(parent=parent, level=level, trace=tr, device_seconds=secs)
