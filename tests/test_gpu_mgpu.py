"""Partitioned (multi-GPU) CUDA kernels on one GPU: P logical ranks driven by one
process through mgpu.LocalComm (collectives as tensor ops; no kernel waits on
another).  Levels, min-id parents and traces must equal the reference's."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MODES = {
    "simd_default": dict(use_simd=True),
    "simd_a14b24": dict(use_simd=True, p=dict(alpha=14, beta=24)),
    "simd_edge": dict(use_simd=True, p=dict(counter_mode="edge")),
    "force_td": dict(use_simd=False, force_direction="top-down"),
    "force_bu": dict(use_simd=True, force_direction="bottom-up"),
}


def trace_array(trace):
    return np.array([[r.layer, 1 if r.direction == "bottom-up" else 0, r.v_f, r.e_f, r.e_u,
                      r.f_value, r.g_value, r.fallback_count, r.gather_count] for r in trace],
                    dtype=np.int64).reshape(-1, 9)


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("name", ["k8", "k10", "u12"])
def test_partitioned_cuda_ranks(cuda, small_golden, golden_hashes, world, name):
    hb = cuda
    from paper_1704_02259_b200.mgpu import CudaRankOps, DistBfs, LocalComm

    rs, adj = small_golden[f"{name}/rs"], small_golden[f"{name}/adj"]
    m = len(adj) // 2
    ranks = [CudaRankOps.from_csr(rs, adj, m, world, r) for r in range(world)]
    db = DistBfs(ranks, LocalComm(world))
    for s in small_golden[f"{name}/sources"][:4]:
        s = int(s)
        for mode, kw in MODES.items():
            p = hb.HeuristicParams(**kw.get("p", {}))
            res = db.bfs(s, p, use_simd=kw["use_simd"], force_direction=kw.get("force_direction"))
            outs = db.outputs()
            par = np.concatenate([o[0] for o in outs])
            lev = np.concatenate([o[1] for o in outs])
            assert np.array_equal(lev, small_golden[f"{name}/{s}/level"]), (name, world, s, mode)
            assert np.array_equal(par, small_golden[f"{name}/{s}/{mode}/parent"]), (name, world, s, mode)
            assert np.array_equal(trace_array(res.trace), small_golden[f"{name}/{s}/{mode}/trace"]), (name, world, s, mode)


def test_partitioned_generate_matches_single_gpu(cuda):
    hb = cuda
    from paper_1704_02259_b200.mgpu import CudaRankOps, DistBfs, LocalComm

    params = hb.GraphParams(scale=14, edgefactor=16, seed=1)
    g = hb.generate_graph(params)
    roots = hb.sample_sources(g, 6, 1)
    for world in (2, 4):
        ranks = [CudaRankOps.generate(params, world, r) for r in range(world)]
        db = DistBfs(ranks, LocalComm(world))
        p = hb.HeuristicParams(alpha=14, beta=24, heuristic="beamer", counter_mode="edge")
        for s in roots:
            ref = hb.bfs(g, int(s), p, device=False)
            res = db.bfs(int(s), p)
            outs = db.outputs()
            assert np.array_equal(np.concatenate([o[1] for o in outs]), ref.level)
            assert np.array_equal(np.concatenate([o[0] for o in outs]), ref.parent)
            assert [r.direction for r in res.trace] == [r.direction for r in ref.trace]


@pytest.mark.parametrize("name", ["k8", "k10", "u12"])
def test_nccl_loop_single_rank(cuda, small_golden, name):
    """The C++ per-layer loop over NCCL (hbfs_mg_bfs) at world size 1: same
    levels, parents and trace as the reference in every mode."""
    hb = cuda
    from paper_1704_02259_b200.mgpu import CudaRankOps, NcclBfs

    rs, adj = small_golden[f"{name}/rs"], small_golden[f"{name}/adj"]
    ops = CudaRankOps.from_csr(rs, adj, len(adj) // 2, 1, 0)
    nb = NcclBfs(ops, 1, 0)
    for s in small_golden[f"{name}/sources"][:4]:
        s = int(s)
        for mode, kw in MODES.items():
            p = hb.HeuristicParams(**kw.get("p", {}))
            res = nb.bfs(s, p, use_simd=kw["use_simd"], force_direction=kw.get("force_direction"))
            par, lev = nb.outputs()[0]
            assert np.array_equal(lev, small_golden[f"{name}/{s}/level"]), (name, s, mode)
            assert np.array_equal(par, small_golden[f"{name}/{s}/{mode}/parent"]), (name, s, mode)
            assert np.array_equal(trace_array(res.trace), small_golden[f"{name}/{s}/{mode}/trace"]), (name, s, mode)
    nb.free()



@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("name", ["k8", "k10", "u12"])
def test_persistent_partition_kernel(cuda, small_golden, world, name, monkeypatch):
    """P ranks of the persistent partition kernel (one launch per layer, the
    C++ loop with device-copy exchanges) on one GPU: levels, min-id parents and
    the trace equal the reference's."""
    hb = cuda
    from paper_1704_02259_b200.mgpu import CudaRankOps, LocalPersistBfs

    if world == 2:  # also the large graphs' deferred level stamping (depth planes + final pass per rank)
        monkeypatch.setenv("HBFS_DEFER_LEVELS_MIN_N", "0")
    rs, adj = small_golden[f"{name}/rs"], small_golden[f"{name}/adj"]
    ranks = [CudaRankOps.from_csr(rs, adj, len(adj) // 2, world, r) for r in range(world)]
    lb = LocalPersistBfs(ranks)
    for s in small_golden[f"{name}/sources"][:4]:
        s = int(s)
        for mode, kw in MODES.items():
            p = hb.HeuristicParams(**kw.get("p", {}))
            res = lb.bfs(s, p, use_simd=kw["use_simd"], force_direction=kw.get("force_direction"))
            outs = lb.outputs()
            par = np.concatenate([o[0] for o in outs])
            lev = np.concatenate([o[1] for o in outs])
            assert np.array_equal(lev, small_golden[f"{name}/{s}/level"]), (name, world, s, mode)
            assert np.array_equal(par, small_golden[f"{name}/{s}/{mode}/parent"]), (name, world, s, mode)
            assert np.array_equal(trace_array(res.trace), small_golden[f"{name}/{s}/{mode}/trace"]), (name, world, s, mode)


def test_persistent_partition_large(cuda, monkeypatch):
    """The large-graph paths (column-blocked and harvest top-down) forced on a
    SCALE 14 graph, P = 1, 2, 4, against the single-GPU traversal."""
    hb = cuda
    from paper_1704_02259_b200.mgpu import CudaRankOps, LocalPersistBfs

    monkeypatch.setenv("HBFS_CB_MIN_N", "1024")
    monkeypatch.setenv("HBFS_CB_MIN_ARCS", "256")
    monkeypatch.setenv("HBFS_HARVEST_MIN_ARCS", "4096")
    params = hb.GraphParams(scale=14, edgefactor=16, seed=1)
    g = hb.generate_graph(params)
    roots = hb.sample_sources(g, 6, 1)
    p = hb.HeuristicParams(alpha=14, beta=24, heuristic="beamer", counter_mode="edge")
    for world in (1, 2, 4):
        lb = LocalPersistBfs([CudaRankOps.generate(params, world, r) for r in range(world)])
        for s in roots:
            ref = hb.bfs(g, int(s), p, device=False)
            res = lb.bfs(int(s), p)
            outs = lb.outputs()
            assert np.array_equal(np.concatenate([o[1] for o in outs]), ref.level), (world, s)
            assert np.array_equal(np.concatenate([o[0] for o in outs]), ref.parent), (world, s)
            assert [r.direction for r in res.trace] == [r.direction for r in ref.trace]


@pytest.mark.parametrize("world", [1, 2, 4])
def test_partitioned_source_sampling_matches_single_gpu(cuda, world):
    """sample_sources_partitioned (order prefix + per-rank degrees, no rank holds
    the whole CSR) picks the reference's roots (harness.py:73-97)."""
    hb = cuda
    from paper_1704_02259_b200.mgpu import CudaRankOps, LocalComm, sample_sources_partitioned

    for params in (hb.GraphParams(scale=14, edgefactor=16, seed=1),
                   hb.GraphParams(scale=10, edgefactor=2, seed=3)):  # many isolated vertices
        g = hb.generate_graph(params)
        ranks = [CudaRankOps.generate(params, world, r) for r in range(world)]
        for count, seed in ((64, 1), (7, 12345)):
            want = hb.sample_sources(g, count, seed)
            got = sample_sources_partitioned(ranks, LocalComm(world), count, seed)
            assert np.array_equal(got, want), (world, count, seed)
        for r in ranks:
            r.free()


def test_exchange_stats_and_pinned_outputs(cuda):
    hb = cuda
    from paper_1704_02259_b200.mgpu import CudaRankOps, LocalPersistBfs

    params = hb.GraphParams(scale=12, edgefactor=16, seed=1)
    g = hb.generate_graph(params)
    s = int(hb.sample_sources(g, 1, 1)[0])
    ref = hb.bfs(g, s, device=False, force_direction="top-down", use_simd=False)
    ranks = [CudaRankOps.generate(params, 2, r) for r in range(2)]
    db = LocalPersistBfs(ranks)
    res = db.bfs(s, force_direction="top-down", use_simd=False)
    outs = db.outputs()
    assert np.array_equal(np.concatenate([o[0] for o in outs]), ref.parent)
    assert np.array_equal(np.concatenate([o[1] for o in outs]), ref.level)
    st = [r.exchange_stats() for r in ranks]
    # top-down layers over few remaining candidates run as local bottom-up sweeps: no records
    assert st[0]["layers"] == len(res.trace) and 0 < st[0]["record_exchanges"] <= len(res.trace)
    assert st[0]["records_sent"] == st[1]["records_received"] > 0


@pytest.mark.parametrize("defer", ["0", str(1 << 40)])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_persistent_partition_deep_traversal(cuda, oracle, world, defer, monkeypatch):
    """More layers than the depth-plane ring holds (32): a 150-vertex path with
    a few chords, through the C++ loop over the persistent partition kernel —
    with levels stamped at discovery and with the deferred stamping of large
    graphs (ring flush of the owned words + final level pass per rank)."""
    hb = cuda
    from paper_1704_02259_b200.mgpu import CudaRankOps, LocalPersistBfs

    monkeypatch.setenv("HBFS_DEFER_LEVELS_MIN_N", defer)

    n = 160
    u = np.arange(0, 149, dtype=np.uint32)
    v = u + 1
    u = np.concatenate([u, np.array([3, 40, 90], dtype=np.uint32)])
    v = np.concatenate([v, np.array([7, 44, 97], dtype=np.uint32)])
    host = oracle.csr_build(u, v, n)
    ranks = [CudaRankOps.from_csr(host.row_starts, host.adjacency, host.in_edges_total, world, r)
             for r in range(world)]
    db = LocalPersistBfs(ranks)
    for s in (0, 75, 149):
        res = db.bfs(s, use_simd=True)
        outs = db.outputs()
        par = np.concatenate([o[0] for o in outs])
        lev = np.concatenate([o[1] for o in outs])
        want_p, want_l, rows = oracle.hybrid_bfs(host, s, use_simd=True)
        assert np.array_equal(lev, want_l), (world, s)
        assert np.array_equal(par, want_p), (world, s)
        assert len(res.trace) == len(rows) and len(rows) > 40
