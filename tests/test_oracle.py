"""Pin the CPU oracle (oracle/hbfs_oracle.c) to the reference's own outputs.

Fixtures in tests/golden/ were produced by the reference package itself
(tests/golden/make_golden.py); these tests prove the restatement is bit-exact
before it is trusted as the checker for the CUDA path.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

MODES = {
    "simd_default": dict(use_simd=True),
    "scalar_default": dict(use_simd=False),
    "simd_a14b24": dict(use_simd=True, alpha=14, beta=24),
    "simd_edge": dict(use_simd=True, counter_mode="edge"),
    "simd_maxpos3": dict(use_simd=True, max_pos=3),
    "force_td": dict(use_simd=False, force_direction="top-down"),
    "force_bu": dict(use_simd=True, force_direction="bottom-up"),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def trace_array(rows):
    return np.array(
        [[r["layer"], r["direction"], r["v_f"], r["e_f"], r["e_u"], r["f_value"], r["g_value"],
          r["fallback_count"], r["gather_count"]] for r in rows], dtype=np.int64).reshape(-1, 9)


def test_mix64_known_values(oracle):
    # splitmix64 finalizer (generator.py:36-44) on fixed inputs
    assert oracle.mix64(0) == 0
    assert oracle.mix64(1) == 0x5692161D100B05E5


@pytest.mark.parametrize("name", ["k8", "k10", "u12", "k11e4"])
def test_small_graphs_against_reference(oracle, small_golden, golden_hashes, name):
    meta = {m["name"]: m for m in golden_hashes["small"]}[name]
    p = meta["params"]
    probs = tuple(p.get("probs", (0.57, 0.19, 0.19, 0.05)))
    u, v = oracle.generate(p["scale"], p["edgefactor"], p["seed"], probs)
    assert np.array_equal(u, small_golden[f"{name}/u"])
    assert np.array_equal(v, small_golden[f"{name}/v"])
    n = 1 << p["scale"]
    g = oracle.csr_build(u, v, n)
    assert np.array_equal(g.row_starts, small_golden[f"{name}/rs"])
    assert np.array_equal(g.adjacency, small_golden[f"{name}/adj"])
    gd = oracle.csr_build(u, v, n, dedup=True)
    assert np.array_equal(gd.row_starts, small_golden[f"{name}/dedup_rs"])
    assert np.array_equal(gd.adjacency, small_golden[f"{name}/dedup_adj"])
    srcs = oracle.sample_sources(g, 8, 1)
    assert np.array_equal(srcs, small_golden[f"{name}/sources"])
    for s in srcs:
        s = int(s)
        _, lev = oracle.bfs_reference(g, s)
        assert np.array_equal(lev, small_golden[f"{name}/{s}/level"])
        for mode, kw in MODES.items():
            par, level, rows = oracle.hybrid_bfs(g, s, **kw)
            assert np.array_equal(par, small_golden[f"{name}/{s}/{mode}/parent"]), (mode, s)
            assert np.array_equal(level, lev), (mode, s)
            assert np.array_equal(trace_array(rows), small_golden[f"{name}/{s}/{mode}/trace"]), (mode, s)
        # F1: every hybrid mode returns the min-id-neighbour-one-level-up tree
        assert np.array_equal(oracle.minid_parents(g, lev, s), small_golden[f"{name}/{s}/simd_default/parent"])


def test_c1_kron_s16_hashes(oracle, golden_hashes):
    rec = golden_hashes["configs"]["C1_kron_s16"]
    u, v = oracle.generate(16, 16, 1)
    assert sha(u) == rec["u_sha"] and sha(v) == rec["v_sha"]
    g = oracle.csr_build(u, v, 1 << 16)
    assert sha(g.row_starts) == rec["rs_sha"] and sha(g.adjacency) == rec["adj_sha"]
    gd = oracle.csr_build(u, v, 1 << 16, dedup=True)
    assert len(gd.adjacency) == rec["dedup_arcs"]
    assert sha(gd.row_starts) == rec["dedup_rs_sha"] and sha(gd.adjacency) == rec["dedup_adj_sha"]
    srcs = oracle.sample_sources(g, 64, 1)
    assert [int(x) for x in srcs] == rec["sources"]
    kw = {"simd_default": MODES["simd_default"], "scalar_default": MODES["scalar_default"],
          "simd_a14b24": MODES["simd_a14b24"]}
    for s in srcs[:16]:
        r = rec["roots"][str(int(s))]
        _, lev = oracle.bfs_reference(g, int(s))
        assert sha(lev) == r["level_sha"]
        for mode, k in kw.items():
            par, level, rows = oracle.hybrid_bfs(g, int(s), **k)
            assert sha(par) == r[mode]["parent_sha"]
            assert trace_array(rows).tolist() == r[mode]["trace"]


@pytest.mark.slow
def test_c2_kron_s20_hashes(oracle, golden_hashes):
    rec = golden_hashes["configs"]["C2_kron_s20"]
    u, v = oracle.generate(20, 16, 1)
    assert sha(u) == rec["u_sha"] and sha(v) == rec["v_sha"]
    g = oracle.csr_build(u, v, 1 << 20)
    assert sha(g.row_starts) == rec["rs_sha"] and sha(g.adjacency) == rec["adj_sha"]
    srcs = oracle.sample_sources(g, 64, 1)
    assert [int(x) for x in srcs] == rec["sources"]
    for s in srcs[:4]:
        r = rec["roots"][str(int(s))]
        par, level, rows = oracle.hybrid_bfs(g, int(s), use_simd=True, alpha=14, beta=24)
        assert sha(level) == r["level_sha"]
        assert sha(par) == r["simd_a14b24"]["parent_sha"]
        assert trace_array(rows).tolist() == r["simd_a14b24"]["trace"]


def test_validator_restatement_faults(oracle):
    # by-hand fault cases of test_acceptance.py:150-203 (rules 2, 3, 5)
    g = oracle.csr_build(np.array([0, 1, 2], np.uint32), np.array([1, 2, 3], np.uint32), 4)
    par, _ = oracle.bfs_reference(g, 0)
    assert oracle.validate_tree(g, 0, par)[0] == 0
    bad = par.copy()
    bad[2], bad[3] = 3, 2
    assert oracle.validate_tree(g, 0, bad)[0] == 3
    gd = oracle.csr_build(np.array([0, 2], np.uint32), np.array([1, 3], np.uint32), 4)
    pd, _ = oracle.bfs_reference(gd, 0)
    pd[2], pd[3] = 3, 2
    assert oracle.validate_tree(gd, 0, pd)[0] == 5
    b2 = par.copy()
    b2[3] = 0
    assert oracle.validate_tree(g, 0, b2) == (2, 3)


def test_byte_model_by_hand():
    """oracle/bytes_model.py on a path 0-1-2 (4-byte row starts), root 0,
    layers TD then BU, against a hand count of SURVEY §8(d)."""
    from oracle.bytes_model import traversal_bytes

    rs = np.array([0, 1, 3, 4])
    adj = np.array([1, 0, 2, 1], dtype=np.uint32)
    level = np.array([0, 1, 2])
    bs, bu = traversal_bytes(rs, adj, level, [0, 1])
    n, W = 3, 1
    init = 8 * n + 12 * W
    # L0 top-down: F={0}: queue 32, rs sector 0, adj sector 0, bitmap sector 0,
    # parent+level sectors of N={1}: 2*32, next queue 32
    td = 32 + 32 + 32 + 32 + 64 + 32
    # L1 bottom-up: U={2} (deg 1, found at position 1 of row [1]... its only
    # entry), rs sector 0, adj sector 0, bitmap sector 0, parent+level 64
    bu_l = 4 * W + 32 + 32 + 32 + 64 + 4 * W
    assert bs == init + td + bu_l
    assert bu == init + (20 * 1 + 4 * 1 + 12 * 1) + (8 * W + 8 * 1 + 4 * 1 + 8 * 1)
