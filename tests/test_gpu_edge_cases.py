"""Edge cases the reference tests (by-hand graphs) on the CUDA path, checked
against the pinned oracle: empty graph, isolated root, self-loops, duplicates,
n not a multiple of 32, MAX_POS boundary, very deep graphs (multi-launch
resume), forced directions, out-of-range roots and validator fault injection."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def graph(hb, pairs, n, dedup=False):
    eu = np.array([p[0] for p in pairs], dtype=np.uint32)
    ev = np.array([p[1] for p in pairs], dtype=np.uint32)
    return hb.from_arrays(eu, ev, n, dedup=dedup), eu, ev


def check_all(hb, oracle, pairs, n, roots=None, **kw):
    g, eu, ev = graph(hb, pairs, n)
    host = oracle.csr_build(eu, ev, n)
    assert np.array_equal(g.row_starts, host.row_starts)
    assert np.array_equal(g.adjacency, host.adjacency)
    for s in (roots if roots is not None else range(n)):
        for simd in (False, True):
            for force in (None, "top-down", "bottom-up"):
                r = hb.bfs(g, s, use_simd=simd, force_direction=force, device=False, **kw)
                par, lev, rows = oracle.hybrid_bfs(host, s, use_simd=simd, force_direction=force)
                assert np.array_equal(r.level, lev), (s, simd, force)
                assert np.array_equal(r.parent, par), (s, simd, force)
                assert len(r.trace) == len(rows)
                for a, b in zip(r.trace, rows):
                    assert (a.v_f, a.e_f, a.e_u, a.f_value, a.g_value, a.fallback_count,
                            a.gather_count) == (b["v_f"], b["e_f"], b["e_u"], b["f_value"],
                                                b["g_value"], b["fallback_count"], b["gather_count"])
    return g


def test_csr_by_hand(cuda):
    hb = cuda
    g, _, _ = graph(hb, [(0, 1), (1, 2)], 3)
    assert list(g.row_starts) == [0, 1, 3, 4] and list(g.adjacency) == [1, 0, 2, 1]
    g, _, _ = graph(hb, [(0, 0)], 2)
    assert list(g.row_starts) == [0, 2, 2] and list(g.adjacency) == [0, 0]
    g, _, _ = graph(hb, [(0, 1), (0, 1)], 2)
    assert list(g.adjacency) == [1, 1, 0, 0] and g.num_arcs == 4
    gd, _, _ = graph(hb, [(0, 1), (0, 1), (2, 2), (1, 0)], 3, dedup=True)
    assert list(gd.row_starts) == [0, 1, 2, 2] and list(gd.adjacency) == [1, 0]
    ge, _, _ = graph(hb, [], 4)
    assert list(ge.row_starts) == [0, 0, 0, 0, 0] and ge.num_arcs == 0 and ge.in_edges_total == 0


def test_empty_and_isolated(cuda, oracle):
    hb = cuda
    check_all(hb, oracle, [], 4)
    check_all(hb, oracle, [(0, 1)], 3)  # vertex 2 isolated


def test_small_shapes(cuda, oracle):
    hb = cuda
    check_all(hb, oracle, [(0, 1), (1, 2)], 3)
    check_all(hb, oracle, [(0, 1), (1, 2), (0, 2)], 3)
    check_all(hb, oracle, [(0, i) for i in range(1, 5)], 5)
    check_all(hb, oracle, [(0, 0), (0, 1), (0, 1), (1, 1), (2, 3)], 37)  # n % 32 != 0
    rng = np.random.default_rng(5)
    pairs = [tuple(int(x) for x in rng.integers(0, 77, 2)) for _ in range(300)]
    check_all(hb, oracle, pairs, 77, roots=range(0, 77, 7))


def test_max_pos_boundary(cuda, oracle):
    # test_acceptance.py:280-321 — vertex 1's only frontier neighbour at position 9
    hb = cuda
    pairs = [(1, v) for v in range(2, 12)]
    g, eu, ev = graph(hb, pairs, 32)
    host = oracle.csr_build(eu, ev, 32)
    for max_pos in (8, 10, 12):
        cfg = hb.VecConfig(max_pos=max_pos)
        r = hb.bfs(g, 11, cfg=cfg, use_simd=True, force_direction="bottom-up", device=False)
        par, lev, rows = oracle.hybrid_bfs(host, 11, use_simd=True, force_direction="bottom-up",
                                           max_pos=max_pos)
        assert r.parent[1] == 11 and np.array_equal(r.parent, par)
        assert r.trace[0].fallback_count == rows[0]["fallback_count"]
        assert (r.trace[0].fallback_count >= 1) == (max_pos == 8)


def test_high_degree_hub_long_rows(cuda, oracle):
    # rows far longer than the per-lane probes: warp-cooperative scan + TD chunking
    hb = cuda
    n = 5000
    pairs = [(0, v) for v in range(1, n)] + [(v, v + 1) for v in range(1, n - 1)]
    pairs += [(4999, v) for v in range(2, 3000, 3)]
    check_all(hb, oracle, pairs, n, roots=[0, 1, 2500, 4999])


@pytest.mark.parametrize("defer", [False, True])
def test_deep_path_resumes_across_launches(cuda, oracle, monkeypatch, defer):
    # 3000 layers > the per-launch trace capacity: exercises the persisted state;
    # with deferred level stamping the 32-plane depth ring wraps ~100 times
    if defer:
        monkeypatch.setenv("HBFS_DEFER_LEVELS_MIN_N", "0")
    hb = cuda
    n = 3000
    pairs = [(i, i + 1) for i in range(n - 1)]
    g, eu, ev = graph(hb, pairs, n)
    host = oracle.csr_build(eu, ev, n)
    r = hb.bfs(g, 0, use_simd=True, device=False)
    par, lev, rows = oracle.hybrid_bfs(host, 0, use_simd=True)
    assert len(r.trace) == len(rows) == n
    assert np.array_equal(r.level, lev) and np.array_equal(r.parent, par)
    assert [t.direction == "bottom-up" for t in r.trace] == [bool(x["direction"]) for x in rows]


@pytest.mark.parametrize("depth", [10, 25, 40])
def test_deferred_levels_full_tiles(cuda, oracle, monkeypatch, depth):
    """levels_kernel paths on full 1024-vertex tiles: all planes in one staged
    batch (depth <= 16), several batches with nothing flushed (16 < depth <
    31), and flushed planes (depth > 30: the per-bit path keeps the levels
    written when a plane was recycled); unreached vertices stay -1."""
    monkeypatch.setenv("HBFS_DEFER_LEVELS_MIN_N", "0")
    n = 6000
    rng = np.random.default_rng(depth)
    spine = list(range(depth + 1))
    pairs = [(spine[i], spine[i + 1]) for i in range(depth)]
    # every other vertex below 5000 hangs off a random spine vertex; 5000.. unreached
    pairs += [(int(rng.integers(0, depth + 1)), v) for v in range(depth + 1, 5000)]
    pairs += [(v, v + 1) for v in range(5000, n - 1, 2)]
    check_all(cuda, oracle, pairs, n, roots=[0, depth // 2, 4000])


@pytest.mark.parametrize("defer", [False, True])
def test_hybrid_bfs_parents_only_out_buffer(cuda, oracle, monkeypatch, defer):
    """hybrid_bfs returns parents only (no level stamping pass) into a reused
    host buffer; a following bfs() on the same workspace still stamps levels."""
    if defer:
        monkeypatch.setenv("HBFS_DEFER_LEVELS_MIN_N", "0")
    hb = cuda
    n = 5000
    rng = np.random.default_rng(7)
    pairs = [(int(a), int(b)) for a, b in rng.integers(0, n, size=(20000, 2))]
    g, eu, ev = graph(hb, pairs, n)
    host = oracle.csr_build(eu, ev, n)
    buf = np.empty(n, dtype=np.uint32)
    for s in (0, 17, 4999):
        par, lev, rows = oracle.hybrid_bfs(host, s, use_simd=True)
        tree, trace = hb.hybrid_bfs(g, s, use_simd=True, out=buf)
        assert tree.parent is buf and np.array_equal(buf, par)
        assert len(trace) == len(rows)
        r = hb.bfs(g, s, use_simd=True, device=False)
        assert np.array_equal(r.level, lev) and np.array_equal(r.parent, par)
    with pytest.raises(ValueError):
        hb.hybrid_bfs(g, 0, out=np.empty(n, dtype=np.int64))
    with pytest.raises(ValueError):
        hb.hybrid_bfs(g, 0, out=np.empty(n - 1, dtype=np.uint32))


def test_errors(cuda):
    hb = cuda
    g, _, _ = graph(hb, [(0, 1), (1, 2)], 3)
    with pytest.raises(IndexError):
        hb.bfs(g, 3)
    with pytest.raises(IndexError):
        hb.hybrid_bfs(g, -1)
    with pytest.raises(ValueError):
        hb.sample_sources(g, 4, 1)
    with pytest.raises(ValueError):
        hb.from_arrays(np.array([0], np.uint32), np.array([5], np.uint32), 3)


def test_validator_faults(cuda):
    # test_acceptance.py:150-203 fault injection -> rules 2, 3, 5 (+1, 4, 6, 7)
    hb = cuda
    g = hb.generate_graph(hb.GraphParams(scale=8, edgefactor=8, seed=11))
    r = hb.bfs(g, 0, device=False)
    assert hb.validate_tree(g, 0, r.parent, r.level, check_minid=True).ok
    par = r.parent.copy()
    v = int(np.flatnonzero(par != hb.NIL)[1])
    nbrs = set(int(x) for x in g.row(v))
    par[v] = next(p for p in range(g.num_vertices) if p not in nbrs and p != v)
    rep = hb.validate_tree(g, 0, par)
    assert not rep.ok and rep.rule == 2 and rep.witness == v
    bad = r.parent.copy()
    bad[0] = 1
    assert hb.validate_tree(g, 0, bad).rule == 1
    gp, _, _ = graph(hb, [(0, 1), (1, 2), (2, 3)], 4)
    tp = hb.bfs(gp, 0, device=False).parent.copy()
    tp[2], tp[3] = 3, 2
    assert hb.validate_tree(gp, 0, tp).rule == 3
    gd, _, _ = graph(hb, [(0, 1), (2, 3)], 4)
    td = hb.bfs(gd, 0, device=False).parent.copy()
    td[2], td[3] = 3, 2
    rep = hb.validate_tree(gd, 0, td)
    assert rep.rule == 5 and rep.witness == 2
    # rule 4: a chord spanning two levels: square 0-1-2-3-0 plus tail, claim 3's parent is 2
    gs, _, _ = graph(hb, [(0, 1), (1, 2), (2, 3), (3, 0)], 4)
    ts = hb.bfs(gs, 0, device=False)
    t4 = ts.parent.copy()
    t4[3] = 2  # 3 now at level 3, but edge (3,0) spans 3 levels
    assert hb.validate_tree(gs, 0, t4).rule == 4
    # rule 6: valid tree but not the min-id parent (triangle + square)
    g6, _, _ = graph(hb, [(0, 1), (0, 2), (1, 3), (2, 3)], 4)
    t6 = hb.bfs(g6, 0, device=False)
    assert t6.parent[3] == 1
    p6 = t6.parent.copy()
    p6[3] = 2
    assert hb.validate_tree(g6, 0, p6).ok
    assert hb.validate_tree(g6, 0, p6, check_minid=True).rule == 6
    lev = t6.level.copy()
    lev[3] = 5
    assert hb.validate_tree(g6, 0, t6.parent, lev).rule == 7


def test_reference_csr_import(cuda, oracle):
    hb = cuda
    u, v = oracle.generate(9, 8, 3)
    host = oracle.csr_build(u, v, 512)
    g = hb.from_csr(host.row_starts, host.adjacency, host.in_edges_total)
    assert g.num_arcs == host.num_arcs and g.in_edges_total == len(u)
    tree, trace = hb.hybrid_bfs(host, 7)  # any object with the reference CsrGraph fields
    par, lev, rows = oracle.hybrid_bfs(host, 7)
    assert np.array_equal(tree.parent, par) and len(trace) == len(rows)


@pytest.mark.parametrize("cb,harvest,by_parent", [(True, False, False), (True, True, False), (False, True, False),
                                                  (True, True, True), (False, True, True)])
def test_top_down_strategies_forced(cuda, oracle, small_golden, golden_hashes, cb, harvest, by_parent):
    """Force the large-layer top-down strategies on the golden small graphs:
    column blocking (every frontier row split into target ranges, normally
    SCALE >= 23 hub layers) and/or the harvest path (fire-and-forget expansion +
    word-order bitmap harvest, normally m_f >= 2^18).  Results must not change."""
    import os

    hb = cuda
    keys = ("HBFS_CB_MIN_N", "HBFS_CB_MIN_ARCS", "HBFS_CB_RANGES", "HBFS_HARVEST_MIN_ARCS",
            "HBFS_DEFER_LEVELS_MIN_N", "HBFS_PARENT_HARVEST_MIN_ARCS")
    old = {k: os.environ.get(k) for k in keys}
    os.environ.update(HBFS_CB_MIN_N="0" if cb else str(1 << 40), HBFS_CB_MIN_ARCS="0",
                      HBFS_CB_RANGES="7", HBFS_HARVEST_MIN_ARCS="0" if harvest else str(1 << 40),
                      HBFS_DEFER_LEVELS_MIN_N="0" if harvest else str(1 << 40),
                      # harvest of the parents (normally >= 2^24 arcs) or of the bitmap
                      HBFS_PARENT_HARVEST_MIN_ARCS="0" if by_parent else str(1 << 40))
    try:
        for meta in golden_hashes["small"]:
            name = meta["name"]
            p = dict(meta["params"])
            if "probs" in p:
                p["probs"] = tuple(p["probs"])
            g = hb.generate_graph(hb.GraphParams(**p))  # fresh workspace reads the knobs
            for s in small_golden[f"{name}/sources"][:4]:
                s = int(s)
                for mode, kw in (("simd_default", dict(use_simd=True)),
                                 ("force_td", dict(use_simd=False, force_direction="top-down"))):
                    r = hb.bfs(g, s, device=False, **kw)
                    assert np.array_equal(r.level, small_golden[f"{name}/{s}/level"]), (name, s, mode)
                    assert np.array_equal(r.parent, small_golden[f"{name}/{s}/{mode}/parent"]), (name, s, mode)
                    # the harvest's counters (next v_f, e_f) drive the trace
                    tr = np.array([[x.layer, 1 if x.direction == "bottom-up" else 0, x.v_f, x.e_f, x.e_u,
                                    x.f_value, x.g_value, x.fallback_count, x.gather_count]
                                   for x in r.trace])
                    assert np.array_equal(tr, small_golden[f"{name}/{s}/{mode}/trace"]), (name, s, mode)
                ra = hb.bfs(g, s, device=False, parent_mode="any", force_direction="top-down")
                assert np.array_equal(ra.level, small_golden[f"{name}/{s}/level"])
                assert hb.validate_tree(g, s, ra.parent, ra.level).ok
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("variant", ["5", "3"])
def test_large_graph_kernel_variant_on_small_graphs(cuda, small_golden, golden_hashes, monkeypatch, variant):
    """The kernel variants of graphs with n >= 2^22 (2 CTAs/SM, 4-vector bottom-up
    probes behind small frontiers; 3 — the default there — or 2 head records per
    lane) forced on the golden small graphs."""
    hb = cuda
    monkeypatch.setenv("HBFS_KERNEL_VARIANT", variant)
    for meta in golden_hashes["small"]:
        name = meta["name"]
        p = dict(meta["params"])
        if "probs" in p:
            p["probs"] = tuple(p["probs"])
        g = hb.generate_graph(hb.GraphParams(**p))  # fresh workspace picks the variant
        for s in small_golden[f"{name}/sources"]:
            s = int(s)
            for mode, kw in (("simd_default", dict(use_simd=True)),
                             ("force_bu", dict(use_simd=True, force_direction="bottom-up")),
                             ("simd_maxpos3", dict(use_simd=True, cfg=hb.VecConfig(max_pos=3)))):
                r = hb.bfs(g, s, device=False, **kw)
                assert np.array_equal(r.level, small_golden[f"{name}/{s}/level"]), (name, s, mode)
                assert np.array_equal(r.parent, small_golden[f"{name}/{s}/{mode}/parent"]), (name, s, mode)
                tr = np.array([[x.layer, 1 if x.direction == "bottom-up" else 0, x.v_f, x.e_f, x.e_u,
                                x.f_value, x.g_value, x.fallback_count, x.gather_count] for x in r.trace])
                assert np.array_equal(tr, small_golden[f"{name}/{s}/{mode}/trace"]), (name, s, mode)


def test_csr_cache_device_roundtrip(cuda, tmp_path):
    hb = cuda
    from paper_1704_02259_b200 import csr

    params = hb.GraphParams(scale=12, edgefactor=16, seed=1)
    g = hb.generate_graph(params)
    csr.save(g, tmp_path / "g.csr", params=params)
    g2 = csr.load(tmp_path / "g.csr")
    assert np.array_equal(g2.row_starts, g.row_starts) and np.array_equal(g2.adjacency, g.adjacency)
    assert g2.in_edges_total == g.in_edges_total
    r1 = hb.bfs(g, 5, device=False)
    r2 = hb.bfs(g2, 5, device=False)
    assert np.array_equal(r1.parent, r2.parent) and np.array_equal(r1.level, r2.level)


def test_run_benchmark_csr_cache(cuda, tmp_path):
    hb = cuda
    params = hb.GraphParams(scale=11, edgefactor=8, seed=4)
    path = tmp_path / "c.csr"
    r1 = hb.run_benchmark(params, mode="simd-hybrid", runs=4, csr_cache=path)
    assert path.exists()
    stamp = path.stat().st_mtime_ns
    r2 = hb.run_benchmark(params, mode="simd-hybrid", runs=4, csr_cache=path)
    assert path.stat().st_mtime_ns == stamp  # reused, not rewritten
    assert [x.source for x in r1.runs] == [x.source for x in r2.runs]
    assert all(x.valid for x in r1.runs + r2.runs)


@pytest.mark.parametrize("name", ["k10", "u12", "k11e4"])
def test_byte_accounting_matches_model(cuda, small_golden, name):
    """The roofline numerator (hbfs_traversal_bytes) equals the
    numpy restatement in oracle/bytes_model.py for every direction mix."""
    hb = cuda
    from oracle.bytes_model import traversal_bytes as model

    rs, adj = small_golden[f"{name}/rs"], small_golden[f"{name}/adj"]
    g = hb.from_csr(rs, adj)
    for s in small_golden[f"{name}/sources"][:3]:
        s = int(s)
        for kw in (dict(), dict(force_direction="top-down"), dict(force_direction="bottom-up")):
            for p in (hb.HeuristicParams(), hb.HeuristicParams(alpha=14, beta=24, heuristic="beamer",
                                                                   counter_mode="edge")):
                r = hb.bfs(g, s, p, device=True, **kw)
                dirs = [1 if x.direction == "bottom-up" else 0 for x in r.trace]
                want = model(rs, adj, r.level.cpu().numpy(), dirs, rs_bytes=8 if g.wide_offsets else 4)
                assert hb.traversal_bytes(g, s, r.level, r.trace) == want, (name, s, kw, p.heuristic)


def test_bfs_out_buffers_checked(cuda):
    """bfs(out=...) refuses buffers the kernel would overrun or misplace."""
    import torch

    hb = cuda
    g, _, _ = graph(hb, [(0, 1), (1, 2), (2, 3)], 40)
    n = g.num_vertices
    good = (torch.empty(n, dtype=torch.int32, device="cuda"), torch.empty(n, dtype=torch.int32, device="cuda"))
    hb.bfs(g, 0, out=good)
    bad = [
        (torch.empty(n - 1, dtype=torch.int32, device="cuda"), good[1]),   # too short
        (good[0], torch.empty(n, dtype=torch.int64, device="cuda")),       # wrong dtype
        (torch.empty(n, dtype=torch.int32), good[1]),                      # CPU tensor
        (torch.empty(2 * n, dtype=torch.int32, device="cuda")[::2], good[1]),  # strided
    ]
    for b in bad:
        with pytest.raises(ValueError):
            hb.bfs(g, 0, out=b)
    with pytest.raises(ValueError):
        hb.bfs(g, 0, device=False, out=(np.empty(n - 1, np.uint32), np.empty(n, np.int32)))
    with pytest.raises(ValueError):
        hb.bfs(g, 0, device=False, out=(np.empty(n, np.int32), np.empty(n, np.int32)))


def test_from_csr_rejects_corrupt(cuda):
    """A foreign CSR (e.g. a damaged cache blob) is refused with ValueError
    instead of being traversed out of bounds."""
    hb = cuda
    rs = np.array([0, 2, 3, 4], dtype=np.int64)
    adj = np.array([1, 2, 0, 0], dtype=np.uint32)
    hb.csr.from_csr(rs, adj).free()
    for r, a in [(rs, np.array([1, 7, 0, 0], np.uint32)),         # id >= n
                 (np.array([0, 3, 2, 4], np.int64), adj),         # decreasing
                 (np.array([1, 2, 3, 4], np.int64), adj)]:        # rs[0] != 0
        with pytest.raises(ValueError):
            hb.csr.from_csr(r, a)


def test_concurrent_calls_on_one_graph(cuda, oracle):
    """hbfs_bfs serialises callers that share a graph workspace: traversals from
    several threads at once all return their own root's exact result."""
    import threading

    hb = cuda
    params = hb.GraphParams(scale=12, edgefactor=16, seed=3)
    g = hb.generate_graph(params)
    host = oracle.HostCsr(g.num_vertices, g.row_starts, g.adjacency, g.in_edges_total)
    roots = [int(x) for x in hb.sample_sources(g, 16, 1)]
    want = {s: oracle.bfs_reference(host, s)[1] for s in roots}
    errors = []

    def work(rs):
        try:
            for _ in range(3):
                for s in rs:
                    r = hb.bfs(g, s, device=False)
                    if not np.array_equal(r.level, want[s]):
                        errors.append(s)
        except Exception as ex:  # pragma: no cover - reported below
            errors.append(repr(ex))

    ts = [threading.Thread(target=work, args=(roots[i::4],)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_imported_graph_released(cuda):
    """as_device_graph frees a reference graph's device copy with the host graph."""
    import gc

    from paper_1704_02259_b200 import csr as C

    hb = cuda

    class RefLike:
        def __init__(self):
            self.row_starts = np.array([0, 1, 2], dtype=np.int64)
            self.adjacency = np.array([1, 0], dtype=np.uint32)
            self.in_edges_total = 1

    h = RefLike()
    tree, _ = hb.hybrid_bfs(h, 0)
    assert list(tree.parent) == [0, 0]
    dg = C.as_device_graph(h)
    assert dg._h is not None and id(h) in C._IMPORTED
    del h
    gc.collect()
    assert dg._h is None
