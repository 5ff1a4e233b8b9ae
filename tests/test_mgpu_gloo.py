"""Multi-rank (1D partition) controller on CPU: world_size 2 and 4 over gloo.

The host logic of paper_1704_02259_b200.mgpu (partitioning, the per-layer
exchange: all-to-all of per-owner counts and all-to-all-v of the top-down
(parent, vertex) records, all-gather of the
next-frontier slices, all-reduce of the switch counters) runs with CPU ranks
(oracle/part_cpu.py) and must reproduce the single-process reference
traversal bit for bit: levels, min-id parents and the trace.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import mgpu_cases


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_partitioned_controller_matches_reference(world, tmp_path, oracle):
    import torch.multiprocessing as mp

    from paper_1704_02259_b200.hybrid import HeuristicParams

    mp.spawn(mgpu_cases.worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for ci, (scale, ef, seed, probs, hk, force) in enumerate(mgpu_cases.CASES):
        u, v = oracle.generate(scale, ef, seed, probs)
        host = oracle.csr_build(u, v, 1 << scale)
        p = HeuristicParams(**hk)
        for pp in parts:  # partitioned root sampling = the reference's, on every rank
            assert np.array_equal(pp[f"{ci}/sources"], oracle.sample_sources(host, 16, 5)), ci
        for ri, root in enumerate(oracle.sample_sources(host, 3, 1)):
            par = np.concatenate([pp[f"{ci}/{ri}/parent"] for pp in parts])
            lev = np.concatenate([pp[f"{ci}/{ri}/level"] for pp in parts])
            want_p, want_l, rows = oracle.hybrid_bfs(
                host, int(root), heuristic=p.heuristic, counter_mode=p.counter_mode,
                alpha=p.alpha, beta=p.beta, use_simd=True, force_direction=force)
            assert np.array_equal(lev, want_l), (ci, ri)
            assert np.array_equal(par, want_p), (ci, ri)
            want_t = np.array([[x["layer"], x["direction"], x["v_f"], x["e_f"], x["e_u"], x["f_value"],
                                x["g_value"], x["fallback_count"], x["gather_count"]] for x in rows])
            for pp in parts:  # every rank saw the same trace
                assert np.array_equal(pp[f"{ci}/{ri}/trace"], want_t), (ci, ri)


def test_partition_ranges_cover_and_align():
    from paper_1704_02259_b200.mgpu import partition

    for n in (64, 100, 1 << 10, 1000):
        for world in (1, 2, 4, 8):
            if n < 32 * world:
                continue
            ranges = [partition(n, world, r)[:2] for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c and a % 32 == 0
