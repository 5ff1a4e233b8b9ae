"""TEST INFRASTRUCTURE — CPU rank for the multi-GPU controller (mgpu.DistBfs).

Implements the same per-rank steps as csrc/part.cu (bottom-up over owned words,
top-down expansion into per-owner (parent, vertex) records, record apply,
frontier absorb) in numpy
on a slice of a host CSR, so the partitioned host logic (exchange order,
padding, counters, decisions) runs under gloo with world_size > 1 on CPU.  The
semantics restated are the reference's layer kernels (_native.pyx:65-204) on an
owned vertex block.  Never used by the product path.
"""

from __future__ import annotations

import numpy as np

INT32_MAX = 0x7FFFFFFF
NIL = 0xFFFFFFFF


def _bits_to_ids(words: np.ndarray, n: int) -> np.ndarray:
    flat = np.unpackbits(words.view(np.uint8), bitorder="little")
    return np.flatnonzero(flat[:n])


class CpuRankOps:
    def __init__(self, row_starts, adjacency, m_edges: int, world: int, rank: int):
        from paper_1704_02259_b200.mgpu import partition

        rs = np.asarray(row_starts, dtype=np.int64)
        self.n = len(rs) - 1
        self.lo, self.hi, _ = partition(self.n, world, rank)
        self.nloc = self.hi - self.lo
        self.rs = rs[self.lo:self.hi + 1] - rs[self.lo]
        self.adj = np.asarray(adjacency, dtype=np.uint32)[rs[self.lo]:rs[self.hi]]
        self.local_arcs = int(len(self.adj))
        self.m_edges = m_edges
        self.W = (self.n + 31) // 32

    def new_tensor(self, size, dtype_name):
        import torch

        return torch.zeros(size, dtype=getattr(torch, dtype_name))

    def degree(self, v: int) -> int:
        if self.lo <= v < self.hi:
            return int(self.rs[v - self.lo + 1] - self.rs[v - self.lo])
        return 0

    def degrees(self, ids) -> np.ndarray:
        ids = np.asarray(ids, dtype=np.int64)
        own = (ids >= self.lo) & (ids < self.hi)
        loc = np.where(own, ids - self.lo, 0)
        return np.where(own, self.rs[loc + 1] - self.rs[loc], 0).astype(np.int64)

    def init(self, root: int):
        self.parent = np.full(self.nloc, NIL, dtype=np.uint32)
        self.level = np.full(self.nloc, -1, dtype=np.int32)
        self.F = np.zeros(self.W, dtype=np.uint32)
        self.F[root >> 5] = np.uint32(1 << (root & 31))
        self.V = self.F.copy()
        if self.lo <= root < self.hi:
            self.parent[root - self.lo] = root
            self.level[root - self.lo] = 0

    def _test(self, words, v):
        return ((words[v >> 5] >> (v & 31)) & 1).astype(bool)

    def bu(self, depth, max_pos, next_slice, ctr):
        nxt = np.zeros(len(next_slice), dtype=np.uint32)
        found = degsum = gathers = fallbacks = 0
        for lv in range(self.nloc):
            v = self.lo + lv
            if (self.V[v >> 5] >> (v & 31)) & 1:
                continue
            s, e = int(self.rs[lv]), int(self.rs[lv + 1])
            if e == s:
                continue
            row = self.adj[s:e]
            hits = np.flatnonzero(self._test(self.F, row))
            deg = e - s
            if len(hits):
                pos = int(hits[0])
                self.parent[lv] = row[pos]
                self.level[lv] = depth + 1
                nxt[lv >> 5] |= np.uint32(1 << (lv & 31))
                found += 1
                degsum += deg
                early = pos < max_pos
                gathers += pos + 1 if early else min(deg, max_pos)
            else:
                early = False
                gathers += min(deg, max_pos)
            fallbacks += int(deg > max_pos and not early)
        next_slice.copy_(self._torch().from_numpy(nxt.view(np.int32)))
        ctr.copy_(self._torch().tensor([found, degsum, gathers, fallbacks], dtype=self._torch().int64))

    def td_expand(self, world, send_counts):
        """Unvisited targets of the owned frontier, each once per owner with
        this rank's min parent candidate (csrc/part.cu kp_td)."""
        from paper_1704_02259_b200.mgpu import partition

        best = {}
        owned = _bits_to_ids(self.F, self.n)
        owned = owned[(owned >= self.lo) & (owned < self.hi)]
        for u in owned:
            lv = u - self.lo
            row = self.adj[self.rs[lv]:self.rs[lv + 1]]
            row = row[~self._test(self.V, row)]
            for v in row.tolist():
                if v not in best or u < best[v]:
                    best[v] = int(u)
        span = partition(self.n, world, 0)[2] * 32
        self._send = [[] for _ in range(world)]
        for v in sorted(best):
            self._send[v // span].append((best[v] << 32) | v)
        send_counts.copy_(self._torch().tensor([len(q) for q in self._send], dtype=self._torch().int64))

    def td_pack(self, records):
        flat = [r for q in self._send for r in q]
        if flat:
            records[: len(flat)].copy_(self._torch().tensor(flat, dtype=self._torch().int64))

    def td_apply(self, depth, records, nrec, next_slice, ctr):
        rec = records.numpy()[:nrec].astype(np.uint64)
        nxt = np.zeros(len(next_slice), dtype=np.uint32)
        best = {}
        for r in rec.tolist():
            v, u = r & 0xFFFFFFFF, r >> 32
            if v not in best or u < best[v]:
                best[v] = u
        deg = 0
        for v, u in best.items():
            lv = v - self.lo
            self.parent[lv] = u
            self.level[lv] = depth + 1
            nxt[lv >> 5] |= np.uint32(1 << (lv & 31))
            deg += int(self.rs[lv + 1] - self.rs[lv])
        next_slice.copy_(self._torch().from_numpy(nxt.view(np.int32)))
        ctr.copy_(self._torch().tensor([len(best), deg, 0, 0], dtype=self._torch().int64))

    def absorb(self, next_full):
        f = next_full.numpy().view(np.uint32)[: self.W].copy()
        self.F = f
        self.V |= f

    def outputs(self):
        return self.parent.copy(), self.level.copy()

    @staticmethod
    def _torch():
        import torch

        return torch
