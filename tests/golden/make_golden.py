"""Generate golden fixtures from the REFERENCE itself (run in the build container).

Imports the reference package read-only from /root/reference/pkg/src, with its
native kernels compiled by oracle/build_ref.py, and records:

* ``small.npz``     — full arrays for small graphs (edges, CSR, sources, levels
                      from ``engine.bfs_reference``, parents + traces from
                      ``hybrid_bfs`` in several modes);
* ``hashes.json``   — SHA-256 digests of the CSR (keep-dup and dedup), the 64
                      sampled roots, per-root levels / parents and the trace
                      tuples for the BASELINE configs C1 (Kron S16), C2 (Kron
                      S20, alpha=14 beta=24 and defaults) and C3 (uniform 2^22).

/root/reference does not exist on the GPU box, so nothing there may run this;
tests read the committed fixtures.  Usage:  python tests/golden/make_golden.py
[--skip-c3]
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from oracle import refnative  # noqa: E402

refnative.load()

import hybfs  # noqa: E402
from hybfs import csr, engine, generator, harness, hybrid  # noqa: E402
from hybfs.lanes import VecConfig  # noqa: E402

assert hybfs.native_available()


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dedup_csr(g):
    n = g.num_vertices
    deg = np.diff(g.row_starts)
    src = np.repeat(np.arange(n, dtype=np.uint64), deg)
    key = (src << np.uint64(32)) | g.adjacency.astype(np.uint64)
    keep = src != g.adjacency.astype(np.uint64)
    if len(key):
        first = np.ones(len(key), dtype=bool)
        first[1:] = key[1:] != key[:-1]
        keep &= first
    rs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src[keep].astype(np.int64), minlength=n), out=rs[1:])
    return rs, g.adjacency[keep]


def trace_tuples(trace):
    return [
        [r.layer, 1 if r.direction == hybrid.BOTTOM_UP else 0, r.v_f, r.e_f, r.e_u,
         r.f_value, r.g_value, r.fallback_count, r.gather_count]
        for r in trace
    ]


MODES = {
    # name: (HeuristicParams kwargs, use_simd, VecConfig kwargs, force)
    "simd_default": ({}, True, {}, None),
    "scalar_default": ({}, False, {}, None),
    "simd_a14b24": ({"alpha": 14, "beta": 24}, True, {}, None),
    "simd_edge": ({"counter_mode": "edge"}, True, {}, None),
    "simd_maxpos3": ({}, True, {"max_pos": 3}, None),
    "force_td": ({}, False, {}, hybrid.TOP_DOWN),
    "force_bu": ({}, True, {}, hybrid.BOTTOM_UP),
}


def run_mode(g, s, mode):
    hp, simd, vc, force = MODES[mode]
    tree, trace = hybrid.hybrid_bfs(
        g, int(s), p=hybrid.HeuristicParams(**hp), cfg=VecConfig(**vc),
        use_simd=simd, engine_name="native", force_direction=force,
    )
    return tree.parent, trace_tuples(trace)


def small_fixtures(out):
    arrays = {}
    meta = []
    specs = [
        ("k8", dict(scale=8, edgefactor=8, seed=2)),
        ("k10", dict(scale=10, edgefactor=16, seed=1)),
        ("u12", dict(scale=12, edgefactor=16, seed=7, probs=(0.25, 0.25, 0.25, 0.25))),
        ("k11e4", dict(scale=11, edgefactor=4, seed=3)),
    ]
    for name, kw in specs:
        p = generator.GraphParams(**kw)
        e = generator.generate(p)
        g = csr.build(e)
        drs, dadj = dedup_csr(g)
        srcs = harness.sample_sources(g, 8, 1)
        arrays[f"{name}/u"] = e.u
        arrays[f"{name}/v"] = e.v
        arrays[f"{name}/rs"] = g.row_starts
        arrays[f"{name}/adj"] = g.adjacency
        arrays[f"{name}/dedup_rs"] = drs
        arrays[f"{name}/dedup_adj"] = dadj
        arrays[f"{name}/sources"] = srcs
        for s in srcs:
            _, lev = engine.bfs_reference(g, int(s))
            arrays[f"{name}/{int(s)}/level"] = lev
            for mode in MODES:
                par, tr = run_mode(g, s, mode)
                arrays[f"{name}/{int(s)}/{mode}/parent"] = par
                arrays[f"{name}/{int(s)}/{mode}/trace"] = np.array(tr, dtype=np.int64).reshape(-1, 9)
        meta.append({"name": name, "params": {k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()},
                     "sources": [int(x) for x in srcs]})
    np.savez_compressed(out, **arrays)
    return meta


def big_config(name, params, modes, runs=64, roots_limit=None):
    t0 = time.time()
    e = generator.generate(params)
    g = csr.build(e)
    drs, dadj = dedup_csr(g)
    srcs = harness.sample_sources(g, runs, params.seed)
    rec = {
        "params": {"scale": params.scale, "edgefactor": params.edgefactor, "seed": params.seed,
                   "probs": list(params.probs)},
        "n": g.num_vertices, "arcs": g.num_arcs, "m": g.in_edges_total,
        "u_sha": sha(e.u), "v_sha": sha(e.v),
        "rs_sha": sha(g.row_starts), "adj_sha": sha(g.adjacency),
        "dedup_arcs": int(len(dadj)), "dedup_rs_sha": sha(drs), "dedup_adj_sha": sha(dadj),
        "max_degree": int(np.diff(g.row_starts).max()),
        "sources": [int(x) for x in srcs],
        "roots": {},
    }
    sel = srcs if roots_limit is None else srcs[:roots_limit]
    for s in sel:
        _, lev = engine.bfs_reference(g, int(s))
        r = {"level_sha": sha(lev), "reached": int((lev >= 0).sum()), "depth": int(lev.max())}
        for mode in modes:
            par, tr = run_mode(g, s, mode)
            r[mode] = {"parent_sha": sha(par), "trace": tr}
        rec["roots"][str(int(s))] = r
    print(f"{name}: {time.time() - t0:.1f}s", flush=True)
    return rec


def main():
    t0 = time.time()
    meta = small_fixtures(os.path.join(HERE, "small.npz"))
    print(f"small fixtures: {time.time() - t0:.1f}s", flush=True)
    hashes = {"small": meta, "configs": {}}
    hashes["configs"]["C1_kron_s16"] = big_config(
        "C1", generator.GraphParams(scale=16, edgefactor=16, seed=1),
        ["simd_default", "scalar_default", "simd_a14b24"])
    hashes["configs"]["C2_kron_s20"] = big_config(
        "C2", generator.GraphParams(scale=20, edgefactor=16, seed=1),
        ["simd_a14b24", "simd_default"])
    if "--skip-c3" not in sys.argv:
        hashes["configs"]["C3_uniform_s22"] = big_config(
            "C3", generator.GraphParams(scale=22, edgefactor=16, seed=1, probs=(0.25,) * 4),
            ["simd_default"], roots_limit=16)
    with open(os.path.join(HERE, "hashes.json"), "w") as fh:
        json.dump(hashes, fh, indent=1)
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
