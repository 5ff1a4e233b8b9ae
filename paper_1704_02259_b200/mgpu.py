"""Multi-GPU hybrid BFS: 1D vertex partition over P ranks.

Rank r owns a contiguous, word-aligned block of vertices with their CSR rows
(global column ids).  The frontier and visited bitmaps are replicated; parent
and level are owned.  Per layer (the controller is the reference's,
hybrid.py:83-175, with the same trace):

* bottom-up: local bottom-up over the owned words against the replicated
  frontier (parents need no communication: rows are local);
* top-down: local expansion of the owned frontier; every unvisited target is
  queued once for its owner with this rank's min parent candidate, the counts
  go **all-to-all** and the 8-byte (parent, vertex) records **all-to-all-v**;
  the owner takes the MIN per vertex (exact min-id parents).  Traffic is
  proportional to the newly reached vertices, never O(n) per layer;
* then **all-gather** of the next-frontier slices (the new replicated frontier,
  also OR-ed into the replicated visited bitmap) and an **all-reduce(SUM)** of
  the four layer counters, so every rank takes the same direction decision.

The per-rank compute is a ``RankOps`` object: ``CudaRankOps`` runs the sm_100a
kernels of ``csrc/part.cu`` (the product); tests also plug in the CPU rank of
``oracle/part_cpu.py`` to cover this host logic with gloo on CPU.  The
communicator is either ``TorchComm`` (one rank per process, torch.distributed
with NCCL on GPUs / gloo on CPU) or ``LocalComm`` (P logical ranks driven by one
process — used to test the partitioned CUDA path on a single GPU; it never runs
kernels that wait on one another).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from .hybrid import BOTTOM_UP, TOP_DOWN, HEURISTICS, COUNTER_MODES, HeuristicParams, LayerTraceRow
from .lanes import VecConfig



def partition(n: int, world: int, rank: int):
    """Owned vertex range [lo, hi) of `rank`: equal word counts per rank."""
    W = (n + 31) // 32
    wper = (W + world - 1) // world
    lo = min(rank * wper * 32, n)
    hi = min((rank + 1) * wper * 32, n)
    return lo, hi, wper


def decide(p: HeuristicParams, cur: int, v_f: int, e_f: int, eu_v: int, eu_e: int, prev_vf: int,
           n: int, force: int):
    """Host restatement of csrc/bfs.cu ``decide`` (reference rule hybrid.py:72-80,
    or Beamer/GAP).  Returns (direction 0/1, f_value, g_value)."""
    gv = n // p.beta
    if p.heuristic == "beamer":
        fv = eu_e // p.alpha
        if force >= 0:
            return force, fv, gv
        if cur == 0:
            return (1 if e_f > fv else 0), fv, gv
        return (0 if (v_f < prev_vf and v_f <= gv) else 1), fv, gv
    e_u = eu_e if p.counter_mode == "edge" else eu_v
    fv = e_u // p.alpha
    if force >= 0:
        return force, fv, gv
    if v_f > fv:
        return 1, fv, gv
    if v_f < gv:
        return 0, fv, gv
    return cur, fv, gv


# ------------------------------------------------------------ communicators

class TorchComm:
    """One rank per process; collectives through torch.distributed."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = dist.get_backend(group)
        self.local_ranks = [self.rank]

    def all_gather(self, slices):
        import torch

        s = slices[0]
        out = torch.empty(s.numel() * self.world, dtype=s.dtype, device=s.device)
        if self.backend == "nccl":
            self.dist.all_gather_into_tensor(out, s, group=self.group)
        else:
            self.dist.all_gather(list(out.chunk(self.world)), s, group=self.group)
        return [out]

    def all_to_all_counts(self, counts):
        """counts[0]: int64[world] sent by this rank to each rank -> int64[world]
        received from each rank."""
        import torch

        out = torch.empty_like(counts[0])
        self.dist.all_to_all_single(out, counts[0], group=self.group)
        return [out]

    def all_to_all_v(self, sendbufs, send_splits, recv_splits):
        import torch

        s = sendbufs[0]
        out = torch.empty(max(1, sum(recv_splits[0])), dtype=s.dtype, device=s.device)
        self.dist.all_to_all_single(out[: sum(recv_splits[0])], s[: sum(send_splits[0])],
                                    recv_splits[0], send_splits[0], group=self.group)
        return [out]

    def all_reduce_sum(self, tensors):
        self.dist.all_reduce(tensors[0], op=self.dist.ReduceOp.SUM, group=self.group)

    def all_reduce_max_float(self, x: float) -> float:
        import torch

        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def barrier(self):
        self.dist.barrier(group=self.group)


class LocalComm:
    """P logical ranks in one process (one GPU): collectives are tensor ops."""

    def __init__(self, world: int):
        self.world = world
        self.rank = 0
        self.local_ranks = list(range(world))

    def all_gather(self, slices):
        import torch

        full = torch.cat(list(slices))
        return [full.clone() for _ in slices]

    def all_to_all_counts(self, counts):
        import torch

        m = torch.stack(list(counts))  # m[src, dst]
        return [m[:, r].clone() for r in range(self.world)]

    def all_to_all_v(self, sendbufs, send_splits, recv_splits):
        import torch

        segs = []  # segs[src][dst]
        for b, sp in zip(sendbufs, send_splits):
            offs = [0]
            for x in sp:
                offs.append(offs[-1] + x)
            segs.append([b[offs[d]:offs[d + 1]] for d in range(self.world)])
        outs = []
        for d in range(self.world):
            parts = [segs[src][d] for src in range(self.world)]
            out = torch.cat(parts) if sum(p.numel() for p in parts) else sendbufs[d].new_empty(1)
            outs.append(out)
        return outs

    def all_reduce_sum(self, tensors):
        tot = tensors[0].clone()
        for t in tensors[1:]:
            tot += t
        for t in tensors:
            t.copy_(tot)

    def all_reduce_max_float(self, x: float) -> float:
        return x

    def barrier(self):
        pass


# -------------------------------------------------------------- CUDA rank

class CudaRankOps:
    """One rank's partition on the current CUDA device (csrc/part.cu)."""

    def __init__(self, handle, device):
        from . import _lib

        self._lib = _lib
        self.lib = _lib.load(require_device=True)
        self.h = handle
        self.device = device
        n, lo, hi, la, m = (C.c_int64() for _ in range(5))
        _lib.check(self.lib.hbfs_part_info(handle, C.byref(n), C.byref(lo), C.byref(hi),
                                           C.byref(la), C.byref(m)))
        self.n, self.lo, self.hi = n.value, lo.value, hi.value
        self.local_arcs, self.m_edges = la.value, m.value
        self.nloc = self.hi - self.lo

    @classmethod
    def generate(cls, params, world: int, rank: int, dedup: bool = False, device=None):
        """Every rank generates the full edge list on its GPU (bit-exact device
        generator) and keeps the rows it owns."""
        import torch

        from . import _lib
        from .generator import thresholds

        lib = _lib.load(require_device=True)
        dev = device or torch.device("cuda", torch.cuda.current_device())
        n, m = params.num_vertices, params.num_edges
        lo, hi, _ = partition(n, world, rank)
        u = torch.empty(m, dtype=torch.int32, device=dev)
        v = torch.empty(m, dtype=torch.int32, device=dev)
        thr = thresholds(params.probs)
        _lib.check(lib.hbfs_generate_edges(params.scale, params.edgefactor,
                                           params.seed & 0xFFFFFFFFFFFFFFFF,
                                           thr.ctypes.data_as(C.c_void_p), int(params.permute_labels),
                                           C.c_void_p(u.data_ptr()), C.c_void_p(v.data_ptr()), 1, None))
        h = C.c_void_p()
        _lib.check(lib.hbfs_part_build(C.c_void_p(u.data_ptr()), C.c_void_p(v.data_ptr()), m, n, lo,
                                       hi, int(dedup), 1, None, C.byref(h)))
        del u, v
        torch.cuda.empty_cache()  # libhbfs allocates with cudaMalloc: hand the edge list's memory back
        return cls(h, dev)

    @classmethod
    def from_csr(cls, row_starts, adjacency, m_edges: int, world: int, rank: int, device=None):
        import torch

        from . import _lib

        lib = _lib.load(require_device=True)
        rs = np.ascontiguousarray(row_starts, dtype=np.int64)
        adj = np.ascontiguousarray(adjacency, dtype=np.uint32)
        n = len(rs) - 1
        lo, hi, _ = partition(n, world, rank)
        h = C.c_void_p()
        _lib.check(lib.hbfs_part_from_csr(rs.ctypes.data_as(C.c_void_p), adj.ctypes.data_as(C.c_void_p),
                                          n, lo, hi, m_edges, None, C.byref(h)))
        return cls(h, device or torch.device("cuda", torch.cuda.current_device()))

    def free(self):
        if self.h is not None:
            self.lib.hbfs_part_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def _s(self):
        return self._lib.current_stream()

    def degree(self, v: int) -> int:
        d = C.c_int64()
        self._lib.check(self.lib.hbfs_part_degree(self.h, v, C.byref(d)))
        return d.value

    def init(self, root: int):
        self._lib.check(self.lib.hbfs_part_init(self.h, root, self._s()))

    def hint_frontier(self, v_f: int):
        self._lib.check(self.lib.hbfs_part_hint_frontier(self.h, int(v_f)))

    def bu(self, depth, max_pos, next_slice, ctr):
        self._lib.check(self.lib.hbfs_part_bu(self.h, depth, max_pos, C.c_void_p(next_slice.data_ptr()),
                                              C.c_void_p(ctr.data_ptr()), self._s()))

    def td_expand(self, world, send_counts):
        self._lib.check(self.lib.hbfs_part_td_expand(self.h, world, C.c_void_p(send_counts.data_ptr()),
                                                     self._s()))

    def td_pack(self, records):
        self._lib.check(self.lib.hbfs_part_td_pack(self.h, C.c_void_p(records.data_ptr()), self._s()))

    def td_apply(self, depth, records, nrec, next_slice, ctr):
        self._lib.check(self.lib.hbfs_part_td_apply(self.h, depth, C.c_void_p(records.data_ptr()), nrec,
                                                    C.c_void_p(next_slice.data_ptr()),
                                                    C.c_void_p(ctr.data_ptr()), self._s()))

    def absorb(self, next_full):
        self._lib.check(self.lib.hbfs_part_absorb(self.h, C.c_void_p(next_full.data_ptr()), self._s()))

    def degrees(self, ids) -> np.ndarray:
        """Degrees of the listed vertices this rank owns (0 for the others)."""
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        deg = np.zeros(len(ids), dtype=np.int64)
        self._lib.check(self.lib.hbfs_part_degrees(self.h, ids.ctypes.data_as(C.c_void_p), len(ids),
                                                   deg.ctypes.data_as(C.c_void_p)))
        return deg

    def exchange_stats(self) -> dict:
        """Exchange volume of the last traversal through the C++ loop."""
        out = (C.c_int64 * 4)()
        self._lib.check(self.lib.hbfs_part_exchange_stats(self.h, out))
        return {"records_sent": out[0], "records_received": out[1], "layers": out[2], "record_exchanges": out[3]}

    def outputs(self):
        """Owned parent/level slices on the host, in pinned arrays reused by
        the next call (the copy runs at the PCIe rate, not through the
        driver's pageable staging)."""
        import torch

        if getattr(self, "_out", None) is None:
            self._out = (torch.empty(max(self.nloc, 1), dtype=torch.int32, pin_memory=True),
                         torch.empty(max(self.nloc, 1), dtype=torch.int32, pin_memory=True))
        tp, tl = self._out
        self._lib.check(self.lib.hbfs_part_outputs(self.h, C.c_void_p(tp.data_ptr()), C.c_void_p(tl.data_ptr()),
                                                   0, self._s()))
        torch.cuda.current_stream().synchronize()
        return tp.numpy()[: self.nloc].view(np.uint32), tl.numpy()[: self.nloc]

    def new_tensor(self, size, dtype_name):
        import torch

        return torch.empty(size, dtype=getattr(torch, dtype_name), device=self.device)


def sample_sources_partitioned(ranks, comm, count: int, seed: int, order_prefix=None) -> np.ndarray:
    """harness.sample_sources (harness.py:73-97) for a partitioned graph: the
    sampling order does not depend on the graph, so its head is generated
    alone (hbfs_source_order_prefix) and filtered by the degrees the ranks
    hold (summed over ranks) — no rank builds the whole CSR.  `ranks`: the
    rank objects this process owns; `comm`: LocalComm / TorchComm;
    `order_prefix(n, seed, k)` (tests: a CPU restatement) defaults to the
    device routine."""
    if order_prefix is None:
        from . import _lib

        lib = _lib.load(require_device=True)

        def order_prefix(n, seed, k):
            ids = np.empty(k, dtype=np.uint32)
            _lib.check(lib.hbfs_source_order_prefix(n, seed & 0xFFFFFFFFFFFFFFFF, k, ids.ctypes.data_as(C.c_void_p)))
            return ids

    r0 = ranks[0]
    n = r0.n
    want = min(n, max(4 * count, 1024))
    while True:
        ids = np.ascontiguousarray(order_prefix(n, seed, want), dtype=np.uint32)
        bufs = []
        for r in ranks:
            t = r.new_tensor(want, "int64")
            t.copy_(_torch_from(r.degrees(ids)))
            bufs.append(t)
        comm.all_reduce_sum(bufs)
        deg = bufs[0].cpu().numpy()
        sel = ids[deg > 0][:count]
        if len(sel) == count:
            return sel
        if want >= n:
            raise ValueError(f"only {len(sel)} vertices with degree >= 1, need {count}")
        want = min(n, want * 4)


def _torch_from(a):
    import torch

    return torch.from_numpy(a)


# ------------------------------------------------------------- controller

@dataclass
class DistResult:
    trace: list
    seconds: float


class DistBfs:
    """Drives the per-layer steps of every rank this process owns (one for
    TorchComm, P for LocalComm) with the same host decisions on all ranks."""

    def __init__(self, ranks, comm):
        self.ranks = list(ranks)
        self.comm = comm
        r0 = self.ranks[0]
        self.n = r0.n
        self.world = comm.world
        _, _, self.wper = partition(self.n, self.world, 0)
        self.W = (self.n + 31) // 32
        arcs = [self._i64([r.local_arcs]) for r in self.ranks]
        comm.all_reduce_sum(arcs)
        self.arcs_global = int(arcs[0][0].item())
        self.m_edges = r0.m_edges

    def _i64(self, vals):
        r0 = self.ranks[0]
        t = r0.new_tensor(len(vals), "int64")
        t.copy_(self._torch().tensor(vals, dtype=self._torch().int64))
        return t

    @staticmethod
    def _torch():
        import torch

        return torch

    def bfs(self, root: int, p: HeuristicParams | None = None, cfg: VecConfig | None = None,
            use_simd: bool = True, force_direction=None) -> DistResult:
        torch = self._torch()
        p = p if p is not None else HeuristicParams()
        cfg = cfg if cfg is not None else VecConfig()
        if not 0 <= root < self.n:
            raise IndexError(f"source {root} out of range [0, {self.n})")
        force = {None: -1, TOP_DOWN: 0, BOTTOM_UP: 1}[force_direction]
        R = self.ranks
        t0 = time.perf_counter()
        for r in R:
            r.init(root)
        degs = [self._i64([r.degree(root)]) for r in R]
        self.comm.all_reduce_sum(degs)
        rdeg = int(degs[0][0].item())
        v_f, e_f, eu_v, eu_e, prev_vf, cur = 1, rdeg, self.n - 1, self.arcs_global - rdeg, 0, 0
        slices = [r.new_tensor(self.wper, "int32") for r in R]
        ctrs = [r.new_tensor(4, "int64") for r in R]
        scounts = [r.new_tensor(self.world, "int64") for r in R]
        trace = []
        layer = 0
        while v_f > 0:
            d, fv, gv = decide(p, cur, v_f, e_f, eu_v, eu_e, prev_vf, self.n, force)
            for s in slices:
                s.zero_()
            tl = time.perf_counter()
            if d == 1:
                for r, s, c in zip(R, slices, ctrs):
                    if hasattr(r, "hint_frontier"):
                        r.hint_frontier(v_f)
                    r.bu(layer, cfg.max_pos, s, c)
            else:
                for r, sc in zip(R, scounts):
                    r.td_expand(self.world, sc)
                rcounts = self.comm.all_to_all_counts(scounts)
                send_splits = [sc.tolist() for sc in scounts]
                recv_splits = [rc.tolist() for rc in rcounts]
                sends = []
                for r, sp in zip(R, send_splits):
                    b = r.new_tensor(max(1, sum(sp)), "int64")
                    r.td_pack(b)
                    sends.append(b)
                recvs = self.comm.all_to_all_v(sends, send_splits, recv_splits)
                for r, rb, rp, s, c in zip(R, recvs, recv_splits, slices, ctrs):
                    r.td_apply(layer, rb, sum(rp), s, c)
            fulls = self.comm.all_gather(slices)
            self.comm.all_reduce_sum(ctrs)
            for r, f in zip(R, fulls):
                r.absorb(f)
            nvf, nef, gat, fb = (int(x) for x in ctrs[0].tolist())
            if d == 0:
                gat, fb = e_f, 0
            if not use_simd:
                gat, fb = 0, 0
            trace.append(LayerTraceRow(
                layer=layer + 1, direction=BOTTOM_UP if d else TOP_DOWN,
                kernel="simd" if use_simd else "scalar", v_f=v_f, e_f=e_f,
                e_u=eu_e if p.counter_mode == "edge" else eu_v, f_value=fv, g_value=gv,
                elapsed=time.perf_counter() - tl, fallback_count=fb, gather_count=gat))
            prev_vf, v_f, e_f = v_f, nvf, nef
            eu_v -= nvf
            eu_e -= nef
            cur = d
            layer += 1
        return DistResult(trace=trace, seconds=time.perf_counter() - t0)

    def outputs(self):
        """Owned (parent, level) of each local rank, in rank order."""
        return [r.outputs() for r in self.ranks]


# ------------------------------------------------ C++ loop over NCCL (GPUs)

class NcclBfs:
    """The per-layer loop of DistBfs in C++ over NCCL (csrc/part.cu
    ``hbfs_mg_bfs``): same steps, same trace, no Python per layer.  One process
    per GPU; the NCCL unique id goes from rank 0 to the others through the
    caller's torch.distributed group (any backend)."""

    def __init__(self, ops: CudaRankOps, world: int, rank: int, group=None):
        import torch  # noqa: F401  (loads torch's libnccl.so.2, which libhbfs then resolves)

        from . import _lib

        self._lib = _lib
        self.ops = ops
        self.lib = ops.lib
        self.world, self.rank = world, rank
        self.n = ops.n
        idbuf = (C.c_uint8 * 128)()
        if rank == 0:
            _lib.check(self.lib.hbfs_nccl_unique_id(idbuf, 128))
        if world > 1:
            import torch
            import torch.distributed as dist

            dev = ops.device if dist.get_backend(group) == "nccl" else "cpu"
            t = torch.tensor(list(bytes(idbuf)), dtype=torch.uint8, device=dev)
            dist.broadcast(t, 0, group=group)
            idbuf = (C.c_uint8 * 128)(*t.cpu().tolist())
        self.h = C.c_void_p()
        _lib.check(self.lib.hbfs_mg_init(idbuf, world, rank, C.byref(self.h)))
        self._rows = (_lib.hbfs_layer_row * 4096)()

    def free(self):
        if self.h:
            self.lib.hbfs_mg_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def bfs(self, root: int, p: HeuristicParams | None = None, cfg: VecConfig | None = None,
            use_simd: bool = True, force_direction=None) -> DistResult:
        from .hybrid import _params

        p = p if p is not None else HeuristicParams()
        cfg = cfg if cfg is not None else VecConfig()
        hp = _params(p, cfg, use_simd, force_direction, "minid")
        nl, ms = C.c_int64(), C.c_float()
        self._lib.check(self.lib.hbfs_mg_bfs(self.h, self.ops.h, int(root), C.byref(hp), self._rows,
                                             len(self._rows), C.byref(nl), C.byref(ms),
                                             self._lib.current_stream()))
        kern = "simd" if use_simd else "scalar"
        trace = [LayerTraceRow(layer=r.layer, direction=BOTTOM_UP if r.direction else TOP_DOWN, kernel=kern,
                               v_f=r.v_f, e_f=r.e_f, e_u=r.e_u, f_value=r.f_value, g_value=r.g_value,
                               elapsed=r.elapsed, fallback_count=r.fallback_count,
                               gather_count=r.gather_count)
                 for r in self._rows[: min(nl.value, len(self._rows))]]
        return DistResult(trace=trace, seconds=ms.value * 1e-3)

    def outputs(self):
        return [self.ops.outputs()]


def run_benchmark_distributed(params, mode: str = "simd-hybrid", heuristic: HeuristicParams | None = None,
                              cfg: VecConfig | None = None, runs: int = 64, allow_isolated: bool = False,
                              source_seed: int | None = None, validate: bool = True):
    """harness.run_benchmark over the 1D partition, one process per GPU
    (torch.distributed initialised with NCCL): rank 0 samples the roots on
    the full graph, every rank traverses its share through NcclBfs, per-root
    time = max over ranks of the device time; trees are all-gathered and
    validated on rank 0 with the device validator.  Returns the
    BenchmarkReport on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    from .csr import generate_graph
    from .harness import (BenchmarkReport, RunResult, _mode_args, harmonic_mean, sample_sources, teps,
                          validate_tree)

    heuristic = heuristic if heuristic is not None else HeuristicParams()
    cfg = cfg if cfg is not None else VecConfig()
    ws, rank = dist.get_world_size(), dist.get_rank()
    dev = torch.device("cuda", torch.cuda.current_device())
    force, use_simd = _mode_args(mode)
    g = None
    roots_t = torch.zeros(runs, dtype=torch.int64, device=dev)
    if rank == 0:
        g = generate_graph(params)
        seed = params.seed if source_seed is None else source_seed
        roots_t.copy_(torch.from_numpy(sample_sources(g, runs, seed, allow_isolated=allow_isolated)
                                       .astype(np.int64)))
        if not validate:
            g.free()
            g = None
    dist.broadcast(roots_t, 0)
    ops = CudaRankOps.generate(params, ws, rank, device=dev)
    nb = NcclBfs(ops, ws, rank)
    n, m = params.num_vertices, params.num_edges
    _, _, wper = partition(n, ws, 0)
    results = []
    for s in roots_t.tolist():
        r = nb.bfs(int(s), heuristic, cfg, use_simd=use_simd, force_direction=force)
        t = torch.tensor([r.seconds], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        par, lev = nb.outputs()[0]
        pad = wper * 32
        loc = torch.full((2, pad), -1, dtype=torch.int32, device=dev)
        loc[0, : len(par)] = torch.from_numpy(par.view(np.int32)).to(dev)
        loc[1, : len(lev)] = torch.from_numpy(lev).to(dev)
        full = torch.empty((ws, 2, pad), dtype=torch.int32, device=dev)
        dist.all_gather_into_tensor(full, loc)
        if rank == 0:
            parent = full[:, 0, :].reshape(-1)[:n].contiguous()
            level = full[:, 1, :].reshape(-1)[:n].contiguous()
            traversed = int((level >= 0).sum().item()) - 1
            secs = float(t.item())
            ok = bool(validate_tree(g, int(s), parent, level)) if validate else True
            results.append(RunResult(source=int(s), seconds=secs, teps=teps(m, secs) if traversed > 0 else 0.0,
                                     valid=ok, trace=r.trace))
    nb.free()
    ops.free()
    if rank != 0:
        return None
    if g is not None:
        g.free()
    positive = [r.teps for r in results if r.teps > 0]
    secs = [r.seconds for r in results]
    return BenchmarkReport(params=params, mode=mode, runs=results,
                           harmonic_mean_teps=harmonic_mean(positive) if positive else 0.0,
                           min_seconds=min(secs), max_seconds=max(secs), mean_seconds=sum(secs) / len(secs),
                           zero_teps_runs=len(results) - len(positive), teps_denominator=m)


class LocalPersistBfs:
    """All P ranks of a partition in this process on one GPU, through the C++
    loop over the persistent partition kernel (``hbfs_mgl_bfs``): the exchange
    steps are device copies.  Tests the multi-GPU kernel path on one GPU."""

    def __init__(self, ranks):
        from . import _lib

        self._lib = _lib
        self.ranks = list(ranks)
        self.lib = self.ranks[0].lib
        self._handles = (C.c_void_p * len(self.ranks))(*[r.h for r in self.ranks])
        self._rows = (_lib.hbfs_layer_row * 4096)()

    def bfs(self, root: int, p: HeuristicParams | None = None, cfg: VecConfig | None = None,
            use_simd: bool = True, force_direction=None) -> DistResult:
        from .hybrid import _params

        p = p if p is not None else HeuristicParams()
        cfg = cfg if cfg is not None else VecConfig()
        hp = _params(p, cfg, use_simd, force_direction, "minid")
        nl, ms = C.c_int64(), C.c_float()
        self._lib.check(self.lib.hbfs_mgl_bfs(self._handles, len(self.ranks), int(root), C.byref(hp), self._rows,
                                              len(self._rows), C.byref(nl), C.byref(ms), self._lib.current_stream()))
        kern = "simd" if use_simd else "scalar"
        trace = [LayerTraceRow(layer=r.layer, direction=BOTTOM_UP if r.direction else TOP_DOWN, kernel=kern,
                               v_f=r.v_f, e_f=r.e_f, e_u=r.e_u, f_value=r.f_value, g_value=r.g_value,
                               elapsed=r.elapsed, fallback_count=r.fallback_count,
                               gather_count=r.gather_count)
                 for r in self._rows[: min(nl.value, len(self._rows))]]
        return DistResult(trace=trace, seconds=ms.value * 1e-3)

    def outputs(self):
        return [r.outputs() for r in self.ranks]
