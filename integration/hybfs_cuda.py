"""Reference-side binding: a ``"cuda"`` engine for the stock ``hybfs`` package.

This is the code INTEGRATION.md tells a reference maintainer to add, as a
module instead of an edit: ``install(hybfs)`` registers the engine on an
imported, unmodified ``hybfs`` (0.1.0) by wrapping the five functions of
``hybfs.engine`` that dispatch on the engine name (engine.py:64-170).  After
that the reference's own controller, ``hybfs.hybrid.hybrid_bfs``
(hybrid.py:83-175), and harness run unchanged with ``engine_name="cuda"``:

* every layer goes through the C ABI (``include/hbfs.h``) via
  ``paper_1704_02259_b200.native`` — ``hbfs_layer_top_down`` for
  ``_native.top_down_layer`` / ``top_down_chunked`` (_native.pyx:65-86,
  :207-239) and ``hbfs_layer_bottom_up`` for ``bottom_up_layer`` /
  ``bottom_up_multiple_set`` (:89-204) — with the graph kept on the device
  (imported once per ``CsrGraph``) and the reference's host bitmaps / parent
  array updated in place exactly as its kernels leave them;
* the counters stay the reference's ``counters_after_layer``
  (bfs_scalar.py:18-26), so the trace is the stock controller's;
* ``engine.bfs_reference(g, s, engine="cuda")`` is ``hbfs_reference_bfs``.

``traverse(g, source, ...)`` is the whole-traversal route (one persistent
kernel, ``hbfs_bfs``) for callers that do not need the per-layer host
bitmaps; it returns the reference's own ``BfsTree`` and ``LayerTraceRow``.

Nothing here runs on the CPU: without libhbfs.so or a CUDA device
``resolve_engine("cuda")`` raises RuntimeError, like ``"native"`` without its
extension (engine.py:72-73).
"""

from __future__ import annotations

import os
import sys
import weakref

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

ENGINE = "cuda"
_graphs: dict = {}  # id(CsrGraph) -> (weakref, rs tensor, adj tensor)


def _device_csr(g):
    """Device copies of a reference CsrGraph's arrays, made once per graph."""
    import torch

    hit = _graphs.get(id(g))
    if hit is not None and hit[0]() is g:
        return hit[1], hit[2]
    rs = torch.from_numpy(np.array(g.row_starts, dtype=np.int64)).cuda()  # writable copies
    adj_np = np.array(g.adjacency, dtype=np.uint32)
    adj = torch.from_numpy(adj_np.view(np.int32)).cuda() if adj_np.size else \
        torch.zeros(1, dtype=torch.int32, device="cuda")
    key = id(g)
    _graphs[key] = (weakref.ref(g), rs, adj)
    weakref.finalize(g, _graphs.pop, key, None)
    return rs, adj


def install(hybfs=None):
    """Register the "cuda" engine on the (imported) stock package; idempotent."""
    if hybfs is None:
        import hybfs  # noqa: F811
    eng = hybfs.engine
    if ENGINE in eng.ENGINES:
        return hybfs
    from paper_1704_02259_b200 import _lib
    from paper_1704_02259_b200 import native as gpu

    counters_after_layer = eng.counters_after_layer
    orig = {name: getattr(eng, name) for name in (
        "resolve_engine", "run_top_down", "run_bottom_up", "run_top_down_chunked",
        "run_bottom_up_multiple_set", "bfs_reference")}

    def resolve_engine(engine: str = "auto", backend: str = "simd") -> str:
        if engine == ENGINE:
            _lib.load(require_device=True)  # RuntimeError without the library / a GPU
            return ENGINE
        return orig["resolve_engine"](engine, backend)

    def run_top_down(g, in_bm, vis, out, tree, engine, stats):
        if engine != ENGINE:
            return orig["run_top_down"](g, in_bm, vis, out, tree, engine, stats)
        rs, adj = _device_csr(g)
        gpu.top_down_layer(rs, adj, in_bm.words, vis.words, out.words, tree.parent, g.num_vertices)
        return counters_after_layer(g, vis, out)

    def run_bottom_up(g, in_bm, vis, out, tree, engine, stats):
        if engine != ENGINE:
            return orig["run_bottom_up"](g, in_bm, vis, out, tree, engine, stats)
        rs, adj = _device_csr(g)
        gpu.bottom_up_layer(rs, adj, in_bm.words, vis.words, out.words, tree.parent, g.num_vertices)
        return counters_after_layer(g, vis, out)

    def run_top_down_chunked(g, in_bm, vis, out, tree, cfg, engine, stats):
        if engine != ENGINE:
            return orig["run_top_down_chunked"](g, in_bm, vis, out, tree, cfg, engine, stats)
        rs, adj = _device_csr(g)
        stats.gather_count += gpu.top_down_chunked(rs, adj, in_bm.words, vis.words, out.words,
                                                   tree.parent, g.num_vertices)
        return counters_after_layer(g, vis, out)

    def run_bottom_up_multiple_set(g, in_bm, vis, out, tree, cfg, engine, stats):
        if engine != ENGINE:
            return orig["run_bottom_up_multiple_set"](g, in_bm, vis, out, tree, cfg, engine, stats)
        rs, adj = _device_csr(g)
        nw = (g.num_vertices + 31) // 32
        dummy = np.zeros(max(nw, 1), dtype=np.uint32)  # rs32/posw/longw: derived on the device
        fb, ga = gpu.bottom_up_multiple_set(rs, adj, in_bm.words, vis.words, out.words, tree.parent,
                                            g.num_vertices, cfg.max_pos, None, dummy, dummy)
        stats.fallback_count += fb
        stats.gather_count += ga
        return counters_after_layer(g, vis, out)

    def bfs_reference(g, source: int, engine: str = "auto"):
        if engine != ENGINE:
            return orig["bfs_reference"](g, source, engine)
        if not 0 <= source < g.num_vertices:
            raise IndexError(f"source {source} out of range [0, {g.num_vertices})")
        rs, adj = _device_csr(g)
        parent, levels = gpu.bfs_reference(rs, adj, g.num_vertices, source)
        return hybfs.frontier.BfsTree(parent=parent, source=source), levels

    eng.ENGINES = tuple(eng.ENGINES) + (ENGINE,)
    eng.resolve_engine = resolve_engine
    eng.run_top_down = run_top_down
    eng.run_bottom_up = run_bottom_up
    eng.run_top_down_chunked = run_top_down_chunked
    eng.run_bottom_up_multiple_set = run_bottom_up_multiple_set
    eng.bfs_reference = bfs_reference
    return hybfs


def traverse(g, source: int, p=None, cfg=None, use_simd: bool = False, force_direction=None):
    """Whole traversal on the device (``hbfs_bfs``: one persistent kernel, the
    direction switch decided on the device) with the reference's signature of
    ``hybrid_bfs`` minus ``engine_name``; returns the stock ``BfsTree`` and
    ``LayerTraceRow`` objects (the reference's heuristic, hybrid.py:62-80)."""
    import hybfs

    import paper_1704_02259_b200 as hb

    p = p if p is not None else hybfs.hybrid.HeuristicParams()
    cfg = cfg if cfg is not None else hybfs.lanes.VecConfig()
    hp = hb.HeuristicParams(alpha=p.alpha, beta=p.beta, counter_mode=p.counter_mode)
    tree, rows = hb.hybrid_bfs(g, int(source), hp, hb.VecConfig(max_pos=cfg.max_pos), use_simd=use_simd,
                               engine_name="cuda", force_direction=force_direction)
    trace = [hybfs.hybrid.LayerTraceRow(
        layer=r.layer, direction=r.direction, kernel=r.kernel, v_f=r.v_f, e_f=r.e_f, e_u=r.e_u,
        f_value=r.f_value, g_value=r.g_value, elapsed=r.elapsed, fallback_count=r.fallback_count,
        gather_count=r.gather_count) for r in rows]
    return hybfs.frontier.BfsTree(parent=np.array(tree.parent, dtype=np.uint32), source=int(source)), trace
