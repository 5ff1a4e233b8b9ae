"""BASELINE INFRASTRUCTURE — the reference's CPU benchmark path, run stock.

bench.py's reference arm (``--impl reference``) and its ``cpu_baseline`` field
time the reference exactly as its own harness does: ``hybfs.harness._run_one``
(harness.py:224-244: perf_counter around ``hybrid.hybrid_bfs``, per-root init
included) of the STOCK package shipped in oracle/_ref (oracle.refpkg) on its
compiled ``_native`` engine (AVX-512 probe when the host has it).

The reference is single-threaded (its ``--threads`` flag is ignored,
cli.py:35-40); to use the host's cores the sample's roots run in concurrent
worker processes forked after the graph is built (the CSR is shared
copy-on-write and never written).  Each worker times its roots with the
stock timer; the step's throughput is roots x m / the slowest worker's summed
traversal time (fork and page-touching stay outside), and the per-traversal
harmonic mean (one core per traversal) is reported beside it.

Graphs: the stock ``generator.generate`` + ``csr.build`` up to SCALE 24; at
SCALE >= 25 the stock generator refuses the size (CapacityError without an
edge budget, generator.py:139-142) and its numpy build needs > 60 GB, so the
C restatement (oracle/hbfs_oracle.c, pinned bit-exact to the stock
generator/CSR at C1-C3 and SCALE 24, and to the device CSR at SCALE 26 by
tests/golden/hashes_s26.json) builds the arrays and the stock ``CsrGraph``
wraps them.

Never imported by the product.
"""

from __future__ import annotations

import os
import pickle
import time

import numpy as np

from . import refpkg


def stock():
    hybfs = refpkg.load()
    if hybfs is None:
        raise RuntimeError("stock hybfs not shipped in oracle/_ref (run oracle/build_ref.py)")
    return hybfs


def stock_graph(scale: int, edgefactor: int = 16, seed: int = 1, probs=(0.57, 0.19, 0.19, 0.05)):
    """(stock CsrGraph, how it was built)."""
    hybfs = stock()
    if scale <= 24:
        p = hybfs.generator.GraphParams(scale=scale, edgefactor=edgefactor, seed=seed, probs=tuple(probs))
        return hybfs.csr.build(hybfs.generator.generate(p)), "stock generator.generate + csr.build"
    from . import oracle as O

    O.build()
    u, v = O.generate(scale, edgefactor, seed, probs)
    h = O.csr_build(u, v, 1 << scale)
    del u, v
    h.row_starts.setflags(write=False)
    h.adjacency.setflags(write=False)
    g = hybfs.csr.CsrGraph(num_vertices=h.num_vertices, num_arcs=h.num_arcs, row_starts=h.row_starts,
                           adjacency=h.adjacency, in_edges_total=h.in_edges_total)
    return g, "C restatement of generate + csr.build (bit-exact, hashes_s26.json), wrapped in stock CsrGraph"


def wrap(num_vertices: int, row_starts, adjacency, m: int):
    """A stock CsrGraph over existing reference-layout arrays."""
    hybfs = stock()
    rs = np.ascontiguousarray(row_starts, dtype=np.int64)
    adj = np.ascontiguousarray(adjacency, dtype=np.uint32)
    return hybfs.csr.CsrGraph(num_vertices=num_vertices, num_arcs=int(rs[-1]), row_starts=rs,
                              adjacency=adj, in_edges_total=int(m))


def sample_sources(g, count: int = 64, seed: int = 1):
    return [int(x) for x in stock().harness.sample_sources(g, count, seed)]


def workers_available() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _touch(g) -> None:
    # map the shared CSR pages in this worker before any timer runs
    int(np.bitwise_xor.reduce(g.adjacency[::1024])) if g.num_arcs else None
    int(g.row_starts[::512].sum())


def _time_some(g, roots, alpha: int, beta: int, mode: str):
    hybfs = stock()
    H = hybfs.hybrid
    _touch(g)
    out = []
    for s in roots:
        tree, _, secs = hybfs.harness._run_one(g, int(s), mode, H.HeuristicParams(alpha=alpha, beta=beta),
                                               hybfs.lanes.VecConfig(), "native")
        out.append((int(s), secs, int(np.count_nonzero(tree.visited_mask())) - 1))
    return out


def time_roots(g, roots, alpha: int, beta: int, workers: int = 1, mode: str = "simd-hybrid"):
    """Time every root with the stock harness timer, `workers` processes at once.

    Returns dict(per_root=[(root, seconds, traversed)], critical_s, workers)."""
    roots = [int(r) for r in roots]
    workers = max(1, min(workers, len(roots)))
    if workers == 1:
        res = _time_some(g, roots, alpha, beta, mode)
        return {"per_root": res, "critical_s": sum(r[1] for r in res), "workers": 1}
    chunks = [roots[i::workers] for i in range(workers)]
    procs = []
    for ch in chunks:
        rfd, wfd = os.pipe()
        pid = os.fork()
        if pid == 0:  # worker: stock traversals only, results pickled back
            os.close(rfd)
            try:
                data = pickle.dumps(("ok", _time_some(g, ch, alpha, beta, mode)))
            except BaseException as ex:  # noqa: BLE001
                data = pickle.dumps(("err", repr(ex)))
            with os.fdopen(wfd, "wb") as fh:
                fh.write(data)
            os._exit(0)
        os.close(wfd)
        procs.append((pid, rfd))
    per_root, crit = [], 0.0
    errors = []
    for pid, rfd in procs:
        with os.fdopen(rfd, "rb") as fh:
            data = fh.read()
        os.waitpid(pid, 0)
        st, res = pickle.loads(data) if data else ("err", "worker died")
        if st != "ok":
            errors.append(res)
            continue
        per_root += res
        crit = max(crit, sum(r[1] for r in res))
    if errors:
        raise RuntimeError(f"reference worker failed: {errors[0]}")
    return {"per_root": per_root, "critical_s": crit, "workers": workers}


def cpu_info() -> dict:
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    nat = stock().engine._native
    d = refpkg.package_dir()
    return {
        "cpu_model": model,
        "host_cores": workers_available(),
        "variant": os.path.basename(d) if d else None,
        "probe_uses_simd": bool(nat.probe_uses_simd()) if nat is not None else None,
    }
