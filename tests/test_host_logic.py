"""Host-side logic of the package (no GPU): parameter validation, the controller
thresholds (reference known answers), TEPS arithmetic, engine selection, the
edge-list file format and the CLI parser."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_1704_02259_b200 as hb
from paper_1704_02259_b200 import generator, hybrid
from paper_1704_02259_b200.frontier import LayerCounters

P = hb.HeuristicParams()


def test_table2_threshold_replay():
    # test_acceptance.py:56-70 / PAPER.md:171-179
    n = 1 << 18
    seq = [262_143, 261_589, 163_864, 86_153, 85_285]
    assert [hb.f_threshold(P, n, LayerCounters(e_u=e)) for e in seq] == [255, 255, 160, 84, 83]
    assert hb.g_threshold(P, n, LayerCounters()) == 4096
    assert hb.g_threshold(P, 64, LayerCounters()) == 1
    assert hb.g_threshold(hb.HeuristicParams(beta=1), 1000, LayerCounters()) == 1000


def test_decide_cases():
    # test_hybrid.py:44-63
    assert hb.decide(P, hb.TOP_DOWN, 554, 1 << 18, LayerCounters(e_u=262_143)) == hb.BOTTOM_UP
    assert hb.decide(P, hb.BOTTOM_UP, 868, 1 << 18, LayerCounters(e_u=85_285)) == hb.BOTTOM_UP
    assert hb.decide(P, hb.BOTTOM_UP, 50, 1 << 18, LayerCounters(e_u=85_285)) == hb.TOP_DOWN
    c = LayerCounters(e_u=10_000_000)
    assert hb.decide(P, hb.BOTTOM_UP, 5000, 1 << 18, c) == hb.BOTTOM_UP
    assert hb.decide(P, hb.TOP_DOWN, 5000, 1 << 18, c) == hb.TOP_DOWN


def test_param_validation():
    with pytest.raises(ValueError):
        hb.HeuristicParams(alpha=0)
    with pytest.raises(ValueError):
        hb.HeuristicParams(counter_mode="mixed")
    with pytest.raises(ValueError):
        hb.HeuristicParams(heuristic="magic")
    with pytest.raises(ValueError):
        hb.VecConfig(max_pos=0)
    with pytest.raises(ValueError):
        hb.VecConfig(backend="avx")
    with pytest.raises(ValueError):
        hb.GraphParams(scale=-1)
    with pytest.raises(ValueError):
        hb.GraphParams(scale=4, probs=(0.5, 0.5, 0.5, 0.5))
    with pytest.raises(ValueError):
        hybrid._params(P, hb.VecConfig(), True, "sideways", "minid")
    with pytest.raises(ValueError):
        hybrid._params(P, hb.VecConfig(), True, None, "random")


def test_engine_selection():
    assert hb.resolve_engine("auto") == "cuda"
    assert hb.resolve_engine("cuda") == "cuda"
    with pytest.raises(RuntimeError):
        hb.resolve_engine("native")
    with pytest.raises(ValueError):
        hb.resolve_engine("fortran")


def test_teps_and_harmonic_mean():
    # test_acceptance.py:360-379 arithmetic
    rng = np.random.default_rng(7)
    for _ in range(200):
        m = int(rng.integers(1, 2**32))
        s = float(rng.uniform(1e-6, 1e3))
        assert hb.teps(m, s) == pytest.approx(m / s, rel=1e-12)
        vals = rng.uniform(1e-3, 1e9, size=int(rng.integers(1, 64))).tolist()
        ref = len(vals) / math.fsum(1.0 / v for v in vals)
        assert hb.harmonic_mean(vals) == pytest.approx(ref, rel=1e-12)
    with pytest.raises(ValueError):
        hb.teps(10, 0.0)
    with pytest.raises(ValueError):
        hb.harmonic_mean([])
    with pytest.raises(ValueError):
        hb.harmonic_mean([1.0, -1.0])


def test_thresholds_python_order():
    t = generator.thresholds((0.57, 0.19, 0.19, 0.05))
    assert t[0] == 0.57 and t[1] == 0.57 + 0.19 and t[2] == (0.57 + 0.19) + 0.19


def test_edge_list_dump_load_roundtrip(tmp_path):
    p = hb.GraphParams(scale=5, edgefactor=2, seed=3)
    e = hb.EdgeList(u=np.arange(64, dtype=np.uint32) % 32, v=np.arange(64, dtype=np.uint32)[::-1] % 32,
                    num_vertices=32, params=p)
    path = tmp_path / "e.bin"
    generator.dump(e, path)
    raw = path.read_bytes()
    assert raw[:8] == b"HBFSEDG1" and len(raw) == 32 + 64 * 16
    back = generator.load(path)
    assert np.array_equal(back.u, e.u) and np.array_equal(back.v, e.v)
    assert back.params.scale == 5 and back.num_vertices == 32


def test_cli_parser():
    from paper_1704_02259_b200 import cli

    a = cli.build_parser().parse_args(["--scale", "12", "--mode", "simd-hybrid", "--heuristic",
                                       "beamer", "--dedup", "--alpha", "14", "--beta", "24"])
    assert a.scale == 12 and a.heuristic == "beamer" and a.dedup and a.alpha == 14
    assert a.engine == "cuda" and a.parent_mode == "minid"


def test_csr_cache_roundtrip(tmp_path, oracle):
    from paper_1704_02259_b200 import csr

    u, v = oracle.generate(9, 8, 3)
    host = oracle.csr_build(u, v, 512)
    p = hb.GraphParams(scale=9, edgefactor=8, seed=3)
    path = tmp_path / "g.csr"
    csr.save(host, path, params=p)
    rs, adj, m, meta = csr.load_arrays(path)
    assert np.array_equal(rs, host.row_starts) and np.array_equal(adj, host.adjacency)
    assert m == len(u) and meta["scale"] == 9 and meta["edgefactor"] == 8 and meta["seed"] == 3
    assert meta["probs"] == (0.57, 0.19, 0.19, 0.05) and not meta["dedup"]
    raw = bytearray(path.read_bytes())
    raw[:8] = b"XXXXXXXX"
    (tmp_path / "bad.csr").write_bytes(bytes(raw))
    with pytest.raises(ValueError):
        csr.load_arrays(tmp_path / "bad.csr")


def test_host_parent_result_arrays(monkeypatch):
    # small results (and HBFS_PINNED_RESULTS=0) are plain pageable uint32 arrays;
    # large ones come from the pinned caching allocator (needs CUDA: GPU tests)
    a = hybrid._host_parent(100)
    assert a.dtype == np.uint32 and a.shape == (100,) and a.flags.c_contiguous
    monkeypatch.setenv("HBFS_PINNED_RESULTS", "0")
    b = hybrid._host_parent(1 << 20)
    assert b.dtype == np.uint32 and b.shape == (1 << 20,) and b.base is None


def test_reference_side_engine_registration():
    """integration/hybfs_cuda.install adds "cuda" to the STOCK hybfs engine
    table; on a host without a GPU, selecting it raises RuntimeError (no CPU
    fallback), while the stock engines keep working."""
    import torch

    from oracle import refpkg

    hybfs = refpkg.load()
    if hybfs is None:
        pytest.skip("oracle/_ref not built (needs /root/reference once)")
    from integration import hybfs_cuda

    hybfs_cuda.install(hybfs)
    hybfs_cuda.install(hybfs)  # idempotent
    assert hybfs.engine.ENGINES.count("cuda") == 1
    assert hybfs.engine.resolve_engine("native") == "native"
    if not torch.cuda.is_available():
        with pytest.raises(RuntimeError):
            hybfs.engine.resolve_engine("cuda")
