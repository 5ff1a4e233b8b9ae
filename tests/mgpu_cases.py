"""Worker for the multi-rank tests (spawned processes; not a test module)."""

from __future__ import annotations

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

CASES = [
    # (scale, edgefactor, seed, probs, heuristic kwargs, force)
    (9, 8, 2, (0.57, 0.19, 0.19, 0.05), dict(), None),
    (9, 8, 2, (0.57, 0.19, 0.19, 0.05), dict(alpha=14, beta=24, heuristic="beamer", counter_mode="edge"), None),
    (10, 4, 7, (0.25, 0.25, 0.25, 0.25), dict(alpha=14, beta=24), None),
    (8, 16, 3, (0.57, 0.19, 0.19, 0.05), dict(), "top-down"),
    (8, 16, 3, (0.57, 0.19, 0.19, 0.05), dict(), "bottom-up"),
]


def worker(rank: int, world: int, port: int, outdir: str, backend: str = "gloo"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group(backend, rank=rank, world_size=world)
    from oracle import oracle as O
    from oracle.part_cpu import CpuRankOps
    from paper_1704_02259_b200.hybrid import HeuristicParams
    from paper_1704_02259_b200.mgpu import DistBfs, TorchComm, sample_sources_partitioned

    out = {}
    for ci, (scale, ef, seed, probs, hk, force) in enumerate(CASES):
        u, v = O.generate(scale, ef, seed, probs)
        host = O.csr_build(u, v, 1 << scale)
        ops = CpuRankOps(host.row_starts, host.adjacency, host.in_edges_total, world, rank)
        db = DistBfs([ops], TorchComm())
        # root sampling without any rank holding all degrees (the order prefix
        # from the oracle: the sampling order with isolated vertices allowed)
        out[f"{ci}/sources"] = sample_sources_partitioned(
            [ops], TorchComm(), 16, 5, order_prefix=lambda n, seed, k: O.sample_sources(host, k, seed, allow_isolated=True))
        for ri, root in enumerate(O.sample_sources(host, 3, 1)):
            res = db.bfs(int(root), HeuristicParams(**hk), use_simd=True, force_direction=force)
            par, lev = db.outputs()[0]
            out[f"{ci}/{ri}/parent"] = par
            out[f"{ci}/{ri}/level"] = lev
            out[f"{ci}/{ri}/trace"] = np.array(
                [[r.layer, 1 if r.direction == "bottom-up" else 0, r.v_f, r.e_f, r.e_u, r.f_value,
                  r.g_value, r.fallback_count, r.gather_count] for r in res.trace], dtype=np.int64)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    dist.destroy_process_group()
