"""The drop-in boundary exercised FROM THE REFERENCE SIDE, and the reference's
own acceptance grid replayed on the CUDA path.

* The stock ``hybfs`` package (the unmodified reference, shipped by
  oracle/build_ref.py into oracle/_ref with its compiled ``_native``) gets the
  ``"cuda"`` engine from ``integration/hybfs_cuda.py`` — the binding
  INTEGRATION.md describes — and its own ``hybrid_bfs`` controller then runs
  against the GPU.  The cases are the reference's engine-equivalence tests
  (test_engine.py:22-68): ``"cuda"`` must be bit-identical to ``"native"`` in
  parents, directions and counters (v_f, e_f, e_u, gathers, fallbacks).
* Criterion 3 of the reference's acceptance suite (test_acceptance.py:117-147):
  every source of every SCALE 4-10 x edgefactor {4, 16} graph, in every mode;
  here levels, parents and traces are held bit-exact to the C oracle (the
  reference only compares levels).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def stock(cuda):
    from oracle import refpkg

    hybfs = refpkg.load()
    assert hybfs is not None, "oracle/_ref must ship the stock hybfs package (oracle/build_ref.py)"
    from integration import hybfs_cuda

    hybfs_cuda.install(hybfs)
    return hybfs


def _gen(hybfs, **kw):
    return hybfs.csr.build(hybfs.generator.generate(hybfs.generator.GraphParams(**kw)))


def test_resolve_engine_cuda(stock):
    eng = stock.engine
    assert "cuda" in eng.ENGINES
    assert eng.resolve_engine("cuda") == "cuda"
    assert eng.resolve_engine("native") == "native"
    with pytest.raises(ValueError):
        eng.resolve_engine("fortran")


def test_reference_bfs_cuda_matches_native(stock):
    """test_engine.py:22-29 with "cuda" in place of "python"."""
    g = _gen(stock, scale=8, edgefactor=8, seed=5)
    for s in (0, 42, 200):
        tn, ln = stock.engine.bfs_reference(g, s, engine="native")
        tc, lc = stock.engine.bfs_reference(g, s, engine="cuda")
        assert np.array_equal(tn.parent, tc.parent)
        assert np.array_equal(ln, lc)
    with pytest.raises(IndexError):
        stock.engine.bfs_reference(g, g.num_vertices, engine="cuda")


@pytest.mark.parametrize("force", [None, "top-down", "bottom-up"])
@pytest.mark.parametrize("use_simd", [False, True])
def test_engines_bit_identical(stock, force, use_simd):
    """test_engine.py:32-44: the stock controller, engine "cuda" vs "native"."""
    H = stock.hybrid
    g = _gen(stock, scale=7, edgefactor=8, seed=9)
    for s in range(0, g.num_vertices, 5):
        tn, trn = H.hybrid_bfs(g, s, use_simd=use_simd, engine_name="native", force_direction=force)
        tc, trc = H.hybrid_bfs(g, s, use_simd=use_simd, engine_name="cuda", force_direction=force)
        assert np.array_equal(tn.parent, tc.parent)
        assert [r.direction for r in trn] == [r.direction for r in trc]
        assert [(r.v_f, r.e_f, r.e_u, r.gather_count, r.fallback_count) for r in trn] == \
            [(r.v_f, r.e_f, r.e_u, r.gather_count, r.fallback_count) for r in trc]


def test_engine_counters_match(stock):
    """test_engine.py:47-56."""
    H = stock.hybrid
    g = _gen(stock, scale=8, edgefactor=16, seed=4)
    for s in (0, 17, 99):
        _, trn = H.hybrid_bfs(g, s, use_simd=True, engine_name="native")
        _, trc = H.hybrid_bfs(g, s, use_simd=True, engine_name="cuda")
        assert len(trn) == len(trc)
        for a, b in zip(trn, trc):
            assert (a.v_f, a.e_f, a.e_u) == (b.v_f, b.e_f, b.e_u)
            assert a.gather_count == b.gather_count
            assert a.fallback_count == b.fallback_count


def test_nondefault_max_pos_matches(stock):
    """test_engine.py:59-68."""
    H = stock.hybrid
    g = _gen(stock, scale=7, edgefactor=8, seed=6)
    for max_pos in (1, 3, 16):
        cfg = stock.lanes.VecConfig(max_pos=max_pos)
        for s in (0, 50):
            tn, trn = H.hybrid_bfs(g, s, cfg=cfg, use_simd=True, engine_name="native")
            tc, trc = H.hybrid_bfs(g, s, cfg=cfg, use_simd=True, engine_name="cuda")
            assert np.array_equal(tn.parent, tc.parent)
            assert [(r.gather_count, r.fallback_count) for r in trn] == \
                [(r.gather_count, r.fallback_count) for r in trc]


def test_stock_harness_runs_on_cuda(stock):
    """The reference's run_benchmark (harness.py:247-296) end to end with the
    cuda engine: every tree passes the reference's own validator."""
    rep = stock.harness.run_benchmark(stock.generator.GraphParams(scale=9, edgefactor=16, seed=2),
                                      mode="simd-hybrid", runs=8, engine_name="cuda")
    assert all(r.valid for r in rep.runs) and rep.harmonic_mean_teps > 0


def test_whole_traversal_route(stock):
    """hybfs_cuda.traverse (hbfs_bfs, one persistent kernel) returns the stock
    types with the stock native engine's parents and trace."""
    from integration import hybfs_cuda

    H = stock.hybrid
    g = _gen(stock, scale=10, edgefactor=16, seed=1)
    for s in (1, 100, 777):
        for simd in (False, True):
            tn, trn = H.hybrid_bfs(g, s, use_simd=simd, engine_name="native")
            tc, trc = hybfs_cuda.traverse(g, s, use_simd=simd)
            assert isinstance(tc, stock.frontier.BfsTree)
            assert np.array_equal(tn.parent, tc.parent)
            key = lambda r: (r.layer, r.direction, r.kernel, r.v_f, r.e_f, r.e_u, r.f_value,
                             r.g_value, r.fallback_count, r.gather_count)
            assert [key(r) for r in trn] == [key(r) for r in trc]


def _rows_equal(trace, rows):
    if len(trace) != len(rows):
        return False
    for a, b in zip(trace, rows):
        if (a.v_f, a.e_f, a.e_u, a.f_value, a.g_value, a.fallback_count, a.gather_count) != \
                (b["v_f"], b["e_f"], b["e_u"], b["f_value"], b["g_value"], b["fallback_count"],
                 b["gather_count"]):
            return False
        if (a.direction == "bottom-up") != bool(b["direction"]):
            return False
    return True


@pytest.mark.parametrize("ef", [4, 16])
def test_acceptance_grid_every_source(cuda, oracle, ef):
    """test_acceptance.py:117-147 on the GPU: every source of SCALE 4..10 at
    this edgefactor; the reference's five variants (scalar/simd hybrid, the
    emulate backend — identical results by construction —, forced TD, forced
    BU) plus Beamer and parent_mode="any".  Levels, parents and traces
    bit-exact against the C oracle; "any" trees pass the Graph500 rules."""
    hb = cuda
    checked = 0
    modes = [
        dict(use_simd=False), dict(use_simd=True), dict(use_simd=False, force_direction="top-down"),
        dict(use_simd=False, force_direction="bottom-up"),
    ]
    beamer = hb.HeuristicParams(alpha=14, beta=24, heuristic="beamer", counter_mode="edge")
    for scale in range(4, 11):
        g = hb.generate_graph(hb.GraphParams(scale=scale, edgefactor=ef, seed=1))
        host = oracle.HostCsr(g.num_vertices, g.row_starts, g.adjacency, g.in_edges_total)
        for s in range(g.num_vertices):
            _, ref_lev = oracle.bfs_reference(host, s)
            for kw in modes:
                r = hb.bfs(g, s, device=False, **kw)
                par, lev, rows = oracle.hybrid_bfs(host, s, **kw)
                assert np.array_equal(r.level, ref_lev), (scale, ef, s, kw)
                assert np.array_equal(r.parent, par), (scale, ef, s, kw)
                assert _rows_equal(r.trace, rows), (scale, ef, s, kw)
                checked += 1
            r = hb.bfs(g, s, beamer, use_simd=True, device=False)
            par, lev, rows = oracle.hybrid_bfs(host, s, heuristic="beamer", counter_mode="edge",
                                               alpha=14, beta=24, use_simd=True)
            assert np.array_equal(r.level, ref_lev) and np.array_equal(r.parent, par), (scale, ef, s)
            assert _rows_equal(r.trace, rows)
            r = hb.bfs(g, s, beamer, use_simd=True, device=False, parent_mode="any")
            assert np.array_equal(r.level, ref_lev)
            assert oracle.validate_tree(host, s, r.parent)[0] == 0, (scale, ef, s)
            checked += 2
        g.free()
    assert checked == 6 * sum(1 << k for k in range(4, 11))
