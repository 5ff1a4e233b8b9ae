"""Graph500-style harness — ``hybfs.harness`` (harness.py:1-334) on the GPU.

Sources, TEPS, harmonic mean and the CSV formats keep the reference's
definitions.  Differences, all on the measurement side:
* the graph is generated and built on the device (``csr.generate_graph``);
* each root's time is the device time of init + traversal (CUDA events around
  the persistent traversal kernel) — the reference times ``hybrid_bfs`` with
  ``perf_counter`` (harness.py:233-244), which also covers init;
* validation runs on the device (``hbfs_validate``), same rules and order.
"""

from __future__ import annotations

import csv
import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import csr as csr_mod
from .csr import as_device_graph
from .frontier import NIL
from .generator import GraphParams
from .hybrid import BOTTOM_UP, TOP_DOWN, HeuristicParams, LayerTraceRow, bfs
from .lanes import VecConfig

MODES = ("scalar-td", "scalar-bu", "scalar-hybrid", "simd-hybrid")
TRACE_FIELDS = "layer,direction,kernel,v_f,e_f,e_u,f,g,seconds,fallbacks,gathers"

RULE_MESSAGES = {
    1: "parent[source] != source",
    2: "parent is not a neighbor",
    3: "parent chain does not reach the source",
    4: "edge spans more than one level",
    5: "visited/reachable mismatch",
    6: "parent is not the minimum-id neighbour one level up",
    7: "level array disagrees with the parent walk",
}


@dataclass
class ValidationReport:
    ok: bool
    rule: int = 0
    witness: int = -1
    message: str = ""

    def __bool__(self) -> bool:
        return self.ok


@dataclass
class RunResult:
    source: int
    seconds: float
    teps: float
    valid: bool
    trace: list = field(default_factory=list)


@dataclass
class BenchmarkReport:
    params: GraphParams
    mode: str
    runs: list
    harmonic_mean_teps: float
    min_seconds: float
    max_seconds: float
    mean_seconds: float
    zero_teps_runs: int
    teps_denominator: int


def sample_sources(g, count: int, seed: int, allow_isolated: bool = False) -> np.ndarray:
    """First ``count`` ids of argsort(mix64(mix64(id+0x5EED)^seed)) with degree >= 1
    (harness.py:73-97), computed on the device."""
    dg = as_device_graph(g)
    n = dg.num_vertices
    if count > n:
        raise ValueError(f"cannot sample {count} distinct vertices from {n}")
    out = np.empty(max(count, 1), dtype=np.uint32)
    lib = _lib.load(require_device=True)
    _lib.check(lib.hbfs_sample_sources(dg.handle, count, seed & 0xFFFFFFFFFFFFFFFF,
                                       int(allow_isolated), out.ctypes.data_as(C.c_void_p)))
    return out[:count]


def validate_tree(g, source: int, tree, level=None, check_minid: bool = False) -> ValidationReport:
    """Graph500 rules 1, 2, 5, 3, 4 (harness.py:129-205) on the device.

    ``tree`` is a BfsTree or a parent array (numpy or torch).  ``level`` (optional)
    is checked against the parent walk (rule 7); ``check_minid`` adds the
    deterministic-parent rule (rule 6)."""
    dg = as_device_graph(g)
    lib = _lib.load(require_device=True)
    parent = getattr(tree, "parent", tree)
    rule = C.c_int32()
    wit = C.c_int64()
    if hasattr(parent, "data_ptr"):
        lp = level.data_ptr() if level is not None else None
        _lib.check(lib.hbfs_validate(dg.handle, source, C.c_void_p(parent.data_ptr()),
                                     C.c_void_p(lp) if lp else None, 1, int(check_minid),
                                     C.byref(rule), C.byref(wit), _lib.current_stream()))
    else:
        par = np.ascontiguousarray(parent, dtype=np.uint32)
        lev = None if level is None else np.ascontiguousarray(level, dtype=np.int32)
        _lib.check(lib.hbfs_validate(dg.handle, source, par.ctypes.data_as(C.c_void_p),
                                     lev.ctypes.data_as(C.c_void_p) if lev is not None else None,
                                     0, int(check_minid), C.byref(rule), C.byref(wit), None))
    r = int(rule.value)
    if r == 0:
        return ValidationReport(True)
    return ValidationReport(False, r, int(wit.value), RULE_MESSAGES.get(r, ""))


def teps(m: int, seconds: float) -> float:
    """Traversed edges per second for an m-edge graph (harness.py:208-212)."""
    if seconds <= 0:
        raise ValueError("duration must be positive")
    return m / seconds


def harmonic_mean(values) -> float:
    """harness.py:215-221."""
    values = list(values)
    if not values:
        raise ValueError("harmonic mean of empty input")
    if any(v <= 0 for v in values):
        raise ValueError("harmonic mean requires positive values")
    return len(values) / sum(1.0 / v for v in values)


def traversal_bytes(g, root: int, level_dev, trace) -> tuple[int, int]:
    """(B_sector, B_useful) of one traversal — SURVEY §8(d) byte model, computed
    on the device from the level array and the layer directions (untimed)."""
    dg = as_device_graph(g)
    lib = _lib.load(require_device=True)
    dirs = np.array([1 if r.direction == BOTTOM_UP else 0 for r in trace], dtype=np.int32)
    bs, bu = C.c_int64(), C.c_int64()
    _lib.check(lib.hbfs_traversal_bytes(dg.handle, root, C.c_void_p(level_dev.data_ptr()),
                                        dirs.ctypes.data_as(C.c_void_p), len(dirs),
                                        C.byref(bs), C.byref(bu), _lib.current_stream()))
    return int(bs.value), int(bu.value)


def _mode_args(mode: str):
    force = {"scalar-td": TOP_DOWN, "scalar-bu": BOTTOM_UP}.get(mode)
    return force, mode == "simd-hybrid"


def run_on_graph(g, sources, mode: str = "simd-hybrid", heuristic: HeuristicParams | None = None,
                 cfg: VecConfig | None = None, validate: bool = True, parent_mode: str = "minid",
                 params: GraphParams | None = None) -> BenchmarkReport:
    """Time one traversal per source on an existing device graph."""
    import torch

    heuristic = heuristic if heuristic is not None else HeuristicParams()
    cfg = cfg if cfg is not None else VecConfig()
    dg = as_device_graph(g)
    n = dg.num_vertices
    m = dg.in_edges_total
    force, use_simd = _mode_args(mode)
    parent = torch.empty(n, dtype=torch.int32, device="cuda")
    level = torch.empty(n, dtype=torch.int32, device="cuda")
    results = []
    for s in sources:
        r = bfs(dg, int(s), heuristic, cfg, use_simd=use_simd, force_direction=force,
                parent_mode=parent_mode, device=True, trace=True, out=(parent, level))
        traversed = int((level >= 0).sum().item()) - 1
        rate = teps(m, r.device_seconds) if traversed > 0 else 0.0
        ok = bool(validate_tree(dg, int(s), parent, level)) if validate else True
        results.append(RunResult(source=int(s), seconds=r.device_seconds, teps=rate, valid=ok,
                                 trace=r.trace))
    positive = [r.teps for r in results if r.teps > 0]
    secs = [r.seconds for r in results]
    return BenchmarkReport(
        params=params, mode=mode, runs=results,
        harmonic_mean_teps=harmonic_mean(positive) if positive else 0.0,
        min_seconds=min(secs), max_seconds=max(secs), mean_seconds=sum(secs) / len(secs),
        zero_teps_runs=len(results) - len(positive), teps_denominator=m,
    )


def run_benchmark(params: GraphParams, mode: str = "scalar-hybrid",
                  heuristic: HeuristicParams | None = None, cfg: VecConfig | None = None,
                  runs: int = 64, allow_isolated: bool = False, engine_name: str = "auto",
                  source_seed: int | None = None, dedup: bool = False,
                  parent_mode: str = "minid", csr_cache=None) -> BenchmarkReport:
    """Generate, build, then time ``runs`` traversals with validation (harness.py:247-296).

    ``csr_cache``: path of a CSR blob (csr.save); reused when its header
    matches ``params``/``dedup``, otherwise (re)written after the build."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    from .engine import resolve_engine

    resolve_engine(engine_name)
    g = _cached_graph(params, dedup, csr_cache)
    seed = params.seed if source_seed is None else source_seed
    sources = sample_sources(g, runs, seed, allow_isolated=allow_isolated)
    rep = run_on_graph(g, sources, mode, heuristic, cfg, validate=True, parent_mode=parent_mode,
                       params=params)
    g.free()
    return rep


def _cached_graph(params: GraphParams, dedup: bool, path):
    import os

    if path is not None and os.path.exists(path):
        try:
            rs, adj, m, meta = csr_mod.load_arrays(path)
            if (meta["scale"], meta["edgefactor"], meta["seed"], meta["probs"], meta["dedup"],
                    meta["permute_labels"]) == (params.scale, params.edgefactor, params.seed,
                                                tuple(params.probs), dedup, params.permute_labels):
                return csr_mod.from_csr(rs, adj, m)
        except ValueError:
            pass
    g = csr_mod.generate_graph(params, dedup=dedup)
    if path is not None:
        csr_mod.save(g, path, params=params, dedup=dedup)
    return g


def write_report_csv(report: BenchmarkReport, path) -> None:
    """source,seconds,teps,valid (harness.py:299-310 format)."""
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        fh.write(
            f"# teps_denominator=undirected_edges m={report.teps_denominator} "
            f"mode={report.mode} scale={report.params.scale} "
            f"edgefactor={report.params.edgefactor} seed={report.params.seed}\n"
        )
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["source", "seconds", "teps", "valid"])
        for r in report.runs:
            w.writerow([r.source, f"{r.seconds:.9f}", f"{r.teps:.3f}", int(r.valid)])


def write_trace_csv(report: BenchmarkReport, path) -> None:
    """Per-layer trace rows (harness.py:313-334 format)."""
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        fh.write(TRACE_FIELDS + "\n")
        w = csv.writer(fh, lineterminator="\n")
        for r in report.runs:
            for row in r.trace:
                w.writerow([row.layer, row.direction, row.kernel, row.v_f, row.e_f, row.e_u,
                            row.f_value, row.g_value, f"{row.elapsed:.9f}", row.fallback_count,
                            row.gather_count])
