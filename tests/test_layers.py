"""Per-layer surface of hybfs._native: the reference's own kernels
recorded in tests/golden/layers.npz (make_layers_golden.py) pin the oracle's
per-layer restatement on CPU and the CUDA implementation (csrc/layer.cu via
paper_1704_02259_b200.native) on the GPU: in-place vis/out/parent, the
chunked and 16-lane counters, and bfs_reference's FIFO-order parents."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN

G = np.load(os.path.join(GOLDEN, "layers.npz"))
NAMES = sorted({k.split("/")[0] for k in G.files})


def cases():
    for name in NAMES:
        for s in G[f"{name}/sources"]:
            s = int(s)
            depth = int(G[f"{name}/{s}/ref_level"].max())
            for d in range(depth + 1):
                yield name, s, d


CASES = list(cases())


def state(name, s, d):
    k = f"{name}/{s}/{d}"
    return (G[f"{name}/rs"], G[f"{name}/adj"], G[k + "/in"], G[k + "/vis"].copy(), G[k + "/out"].copy(),
            G[k + "/parent"].copy(), len(G[f"{name}/rs"]) - 1)


def posw_longw(rs, mp):
    deg = np.diff(rs)
    n = len(deg)
    nw = (n + 31) // 32

    def bits(m):
        w = np.zeros(nw * 32, dtype=np.uint8)
        w[:n] = m
        return np.packbits(w, bitorder="little").view(np.uint32).copy()

    return bits(deg > 0), bits(deg > mp)


# ------------------------------------------------------------------ CPU: oracle

def test_oracle_layers_match_reference_kernels(oracle):
    for name, s, d in CASES:
        k = f"{name}/{s}/{d}"
        rs, adj, inw, vis, out, par, n = state(name, s, d)
        g = oracle.td_layer(rs, adj, n, inw, vis, out, par)
        for arr, key in ((vis, "vis"), (out, "out"), (par, "parent")):
            assert np.array_equal(arr, G[f"{k}/td/{key}"]), (k, "td", key)
        assert g == int(G[f"{k}/tdc/gathers"])
        rs, adj, inw, vis, out, par, n = state(name, s, d)
        oracle.bu_layer(rs, adj, n, inw, vis, out, par)
        for arr, key in ((vis, "vis"), (out, "out"), (par, "parent")):
            assert np.array_equal(arr, G[f"{k}/bu/{key}"]), (k, "bu", key)
        for mp in (1, 3, 8, 16):
            rs, adj, inw, vis, out, par, n = state(name, s, d)
            posw, longw = posw_longw(rs, mp)
            fb, ga = oracle.bu_multiple_set(rs, adj, n, mp, posw, longw, inw, vis, out, par)
            k2 = f"{k}/bums{mp}"
            for arr, key in ((vis, "vis"), (out, "out"), (par, "parent")):
                assert np.array_equal(arr, G[f"{k2}/{key}"]), (k2, key)
            assert [fb, ga] == G[f"{k2}/counters"].tolist(), k2


def test_oracle_bfs_reference_matches_reference_kernel(oracle):
    for name in NAMES:
        rs = G[f"{name}/rs"]
        g = oracle.HostCsr(len(rs) - 1, rs, G[f"{name}/adj"], 0)
        for s in G[f"{name}/sources"]:
            par, lev = oracle.bfs_reference(g, int(s))
            assert np.array_equal(lev, G[f"{name}/{int(s)}/ref_level"])
            assert np.array_equal(par, G[f"{name}/{int(s)}/ref_parent"])


def test_native_module_needs_the_gpu():
    """No CPU path: without a device the per-layer calls raise."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_1704_02259_b200 import native

    rs, adj, inw, vis, out, par, n = state(*CASES[0])
    with pytest.raises(RuntimeError):
        native.top_down_layer(rs, adj, inw, vis, out, par, n)
    assert native.probe_uses_simd() is True


# ------------------------------------------------------------------ GPU: CUDA

@pytest.mark.gpu
@pytest.mark.parametrize("on_device", [False, True])
def test_cuda_layers_match_reference_kernels(cuda, on_device):
    import torch

    from paper_1704_02259_b200 import native

    def dev(a):
        return torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).cuda() if on_device else a

    def host(t, like):
        return t.cpu().numpy().view(like.dtype) if on_device else t

    for name, s, d in CASES:
        k = f"{name}/{s}/{d}"
        for kern in ("td", "tdc", "bu"):
            rs, adj, inw, vis, out, par, n = state(name, s, d)
            args = [dev(x) for x in (rs, adj, inw, vis, out, par)]
            if kern == "td":
                native.top_down_layer(*args, n)
            elif kern == "tdc":
                assert native.top_down_chunked(*args, n) == int(G[f"{k}/tdc/gathers"]), k
            else:
                native.bottom_up_layer(*args, n)
            for t, like, key in ((args[3], vis, "vis"), (args[4], out, "out"), (args[5], par, "parent")):
                assert np.array_equal(host(t, like), G[f"{k}/{kern}/{key}"]), (k, kern, key)
        for mp in (1, 3, 8, 16):
            rs, adj, inw, vis, out, par, n = state(name, s, d)
            posw, longw = posw_longw(rs, mp)
            args = [dev(x) for x in (rs, adj, inw, vis, out, par)]
            fb, ga = native.bottom_up_multiple_set(*args, n, mp, rs.astype(np.int32), posw, longw)
            k2 = f"{k}/bums{mp}"
            assert [fb, ga] == G[f"{k2}/counters"].tolist(), k2
            for t, like, key in ((args[3], vis, "vis"), (args[4], out, "out"), (args[5], par, "parent")):
                assert np.array_equal(host(t, like), G[f"{k2}/{key}"]), (k2, key)


@pytest.mark.gpu
def test_cuda_bfs_reference_fifo_parents(cuda):
    from paper_1704_02259_b200 import engine, native
    from paper_1704_02259_b200.csr import from_csr

    for name in NAMES:
        rs, adj = G[f"{name}/rs"], G[f"{name}/adj"]
        n = len(rs) - 1
        for s in G[f"{name}/sources"]:
            par, lev = native.bfs_reference(rs, adj, n, int(s))
            assert np.array_equal(lev, G[f"{name}/{int(s)}/ref_level"])
            assert np.array_equal(par, G[f"{name}/{int(s)}/ref_parent"])
        g = from_csr(rs, adj)
        tree, lev = engine.bfs_reference(g, int(G[f"{name}/sources"][0]))
        assert np.array_equal(tree.parent, G[f"{name}/{int(G[f'{name}/sources'][0])}/ref_parent"])
        with pytest.raises(IndexError):
            engine.bfs_reference(g, n)


def _graph(pairs, n):
    """Undirected keep-dup CSR from an edge list (csr.py:46-74 layout)."""
    src = np.array([a for a, b in pairs] + [b for a, b in pairs], dtype=np.uint64)
    dst = np.array([b for a, b in pairs] + [a for a, b in pairs], dtype=np.uint64)
    order = np.argsort((src << np.uint64(32)) | dst, kind="stable")
    adj = dst[order].astype(np.uint32)
    rs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src.astype(np.int64), minlength=n), out=rs[1:])
    return rs, adj


def _fresh(n, frontier):
    nw = (n + 31) // 32
    inw = np.zeros(nw, dtype=np.uint32)
    for f in frontier:
        inw[f >> 5] |= np.uint32(1 << (f & 31))
    par = np.full(n, 0xFFFFFFFF, dtype=np.uint32)
    par[frontier[0]] = frontier[0]
    return inw, inw.copy(), np.zeros(nw, dtype=np.uint32), par


@pytest.mark.gpu
def test_cuda_layer_known_answers(cuda):
    """The reference's hand-made cases (test_bfs_scalar.py / test_bfs_vector.py)."""
    from paper_1704_02259_b200 import native

    # 20-leaf star: chunked top-down claims every leaf, gathers 16 + 4
    rs, adj = _graph([(0, i) for i in range(1, 21)], 21)
    inw, vis, out, par = _fresh(21, [0])
    assert native.top_down_chunked(rs, adj, inw, vis, out, par, 21) == 20
    assert all(par[v] == 0 for v in range(1, 21))
    # first frontier entry of the sorted row wins: 3 ~ {1, 2} -> parent 1
    rs, adj = _graph([(0, 1), (0, 2), (3, 2), (3, 1)], 4)
    inw, vis, out, par = _fresh(4, [1, 2])
    native.bottom_up_layer(rs, adj, inw, vis, out, par, 4)
    assert par[3] == 1
    # vertex 20's only frontier neighbour at row position 10: fallback at
    # max_pos 8, probe alone at max_pos 11
    rs, adj = _graph([(20, v) for v in range(1, 12)] + [(0, 11)], 21)
    assert list(adj[rs[20]:rs[21]]).index(11) == 10
    for mp, want_fb in ((8, True), (11, False)):
        inw, vis, out, par = _fresh(21, [11])
        posw, longw = posw_longw(rs, mp)
        fb, ga = native.bottom_up_multiple_set(rs, adj, inw, vis, out, par, 21, mp, None, posw, longw)
        assert par[20] == 11
        assert (fb >= 1) == want_fb
    # dtype contract of the Cython buffers
    with pytest.raises(ValueError):
        native.bottom_up_layer(rs.astype(np.int32), adj, inw, vis, out, par, 21)


def test_native_argument_checks_on_cpu():
    """Buffer-length and dtype contract of the _native surface (checked before
    any device work, so it holds on the CPU too)."""
    from paper_1704_02259_b200 import native

    rs, adj, inw, vis, out, par, n = state(*CASES[0])
    with pytest.raises(ValueError):
        native.top_down_layer(rs[:-1], adj, inw, vis, out, par, n)  # rs shorter than n + 1
    with pytest.raises(ValueError):
        native.bottom_up_layer(rs, adj, inw[:0], vis, out, par, n)  # frontier bitmap too short
    with pytest.raises(ValueError):
        native.top_down_chunked(rs, adj, inw, vis, out, par[:-1], n)  # parent too short
    with pytest.raises(ValueError):
        native.bottom_up_layer(rs, adj[:-1], inw, vis, out, par, n)  # adjacency shorter than rs[n]
    with pytest.raises(ValueError):
        native.bottom_up_multiple_set(rs, adj, inw, vis, out, par, n, 0, None, vis, vis)  # max_pos < 1
    with pytest.raises(ValueError):
        native.bfs_reference(rs, adj[:-1], n, 0)


def test_engine_bfs_reference_range_check_on_cpu():
    from paper_1704_02259_b200 import engine

    class G:  # the attributes engine.bfs_reference reads before any device work
        num_vertices = 4
        row_starts = np.zeros(5, dtype=np.int64)
        adjacency = np.zeros(0, dtype=np.uint32)

    with pytest.raises(IndexError):
        engine.bfs_reference(G(), 4)
    with pytest.raises(RuntimeError):
        engine.bfs_reference(G(), 0, engine="native")  # the reference's CPU engine name
