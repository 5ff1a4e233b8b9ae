// Multi-GPU hybrid BFS: one rank's share of a 1D vertex partition.
//
// Rank r owns vertices [lo, hi) (word aligned) and holds their CSR rows with
// global column ids.  The frontier bitmap F and the visited bitmap V are
// replicated (n bits each); parent/level are owned-only.  Per layer the host
// (paper_1704_02259_b200/mgpu.py) runs one of
//   bottom-up:  hbfs_part_bu        -> next-frontier slice of the owned words
//                                      (the persistent kernel's tile code,
//                                      bfs.cu part_bu_launch)
//   top-down:   hbfs_part_td_expand -> min parent candidate per unvisited
//                                      target + a touch bitmap (fire-and-
//                                      forget reductions), scanned into
//                                      record counts per owner
//               [all-to-all of the counts]
//               hbfs_part_td_pack   -> 8-byte (parent, vertex) records packed
//                                      by owner
//               [NCCL all-to-all-v of the records]
//               hbfs_part_td_apply  -> owned parents/levels + next slice
// then [NCCL all-gather of the slices] and hbfs_part_absorb (F = next,
// V |= next), plus an all-reduce of the four layer counters.  Top-down traffic
// is 8 bytes per (rank, newly reached vertex) pair, not O(n) per layer.
// Parents are the global min-id neighbour one level up: bottom-up
// takes the first frontier hit in the sorted row, top-down the MIN over every
// rank's arcs (each rank pre-reduces its own, the owner reduces the records).
// Replaces, for P > 1, the same reference functions as bfs.cu.
#include <cub/cub.cuh>

#include "common.cuh"

namespace hbfs {

struct Part {
    int64_t n = 0, lo = 0, hi = 0, nloc = 0, W = 0, wlo = 0, wloc = 0;
    int64_t arcs = 0;         // local arcs
    int64_t m_edges = 0;      // global TEPS denominator
    DevBuf rs;                // uint64[nloc + 1], local offsets
    DevBuf adj;               // uint32[arcs + 8], global ids
    DevBuf F, V;              // uint32[W] replicated
    DevBuf parent, level;     // owned
    DevBuf q;                 // uint32[nloc] owned frontier queue
    DevBuf seg_u, seg_k;      // long-row segments (row, first arc), <= arcs/4096 + nloc/1024
    DevBuf pieces, rcnt;      // range-ordered pieces (Piece); per-range counts/cursors
    int64_t nseg_cap = 0;
    int ranges = 1;
    DevBuf scratch;           // counters etc.
    DevBuf posw;              // uint32[wloc] deg > 0 bits of the owned vertices
    DevBuf hd, pre;           // head records of the owned rows, rank order + per-word prefix (common.cuh)
    int64_t n_pos = 0;        // owned vertices with degree > 0
    DevBuf bu_scratch;        // part_bu_launch scratch (Ctl)
    int64_t fhint = -1;       // global frontier size of the next bottom-up layer (-1: unknown)
    // top-down exchange state (all kept clean between layers)
    DevBuf cand;              // int32[n]  min parent candidate per target (INT32_MAX = none)
    DevBuf touch;             // uint32[W] target already queued this layer
    DevBuf candown;           // int32[nloc] min over the received records
    DevBuf wcnt, wexcl;       // uint32[W + 1] touch-word popcounts and their exclusive prefix
    DevBuf scan_tmp;          // CUB scan scratch
    size_t scan_bytes = 0;
    int world = 0;            // partition the queues were sized for
    int64_t span = 0;         // vertices per owner block (word aligned)
    void *trav = nullptr;     // persistent-kernel traversal state (bfs.cu part_trav_*)
    DevBuf recs_s, recs_r, acnt;  // records out / in, apply counters
    DevBuf counts_dev;        // int64[2 * world] record counts sent / received
    unsigned long long *h_acnt = nullptr;  // pinned: the layer's counter totals (after the layer's stream sync)
    DevBuf lay;                            // device: the layer's counter totals, uint64[4]
    int64_t stat[4] = {0, 0, 0, 0};        // last traversal: records sent, received, layers, record exchanges
    size_t cap_s = 0, cap_r = 0;
    ~Part() {
        if (trav) part_trav_free(trav);
        if (h_acnt) cudaFreeHost(h_acnt);
    }
};

static inline int pgrid(int64_t items, int block = 256) {
    int64_t g = (items + block - 1) / block;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

#define PSTRIDE(i, N) \
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (N); i += (int64_t)gridDim.x * blockDim.x)

// Arcs whose source is owned: key = (local src << sb) | global dst.  key == null
// only counts (first pass sizes the buffer exactly).
__global__ void kp_arc_keys(int64_t m, int sb, int64_t lo, int64_t hi, const uint32_t *u,
                            const uint32_t *v, uint64_t *key, unsigned long long *cnt) {
    unsigned long long local = 0;
    PSTRIDE(e, m) {
        const uint64_t a = u[e], b = v[e];
        const bool oa = (int64_t)a >= lo && (int64_t)a < hi, ob = (int64_t)b >= lo && (int64_t)b < hi;
        if (!key) {
            local += (unsigned long long)oa + (unsigned long long)ob;
            continue;
        }
        if (oa) key[atomicAdd(cnt, 1ull)] = ((a - lo) << sb) | b;
        if (ob) key[atomicAdd(cnt, 1ull)] = ((b - lo) << sb) | a;
    }
    if (!key && local) atomicAdd(cnt, local);
}

__global__ void kp_dedup_flags(int64_t k, int sb, int64_t lo, const uint64_t *key, uint8_t *keep) {
    const uint64_t mask = (uint64_t(1) << sb) - 1;
    PSTRIDE(i, k) {
        const uint64_t x = key[i];
        const bool self = (int64_t)((x >> sb) + lo) == (int64_t)(x & mask);
        keep[i] = !(self || (i > 0 && key[i - 1] == x));
    }
}

__global__ void kp_adj(int64_t k, int sb, const uint64_t *key, uint32_t *adj) {
    const uint64_t mask = (uint64_t(1) << sb) - 1;
    PSTRIDE(i, k) adj[i] = (uint32_t)(key[i] & mask);
}

__global__ void kp_rs(int64_t nloc, int64_t k, int sb, const uint64_t *key, uint64_t *rs) {
    PSTRIDE(v, nloc + 1) {
        const uint64_t target = (uint64_t)v << sb;
        int64_t lo = 0, hi = k;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (key[mid] < target) lo = mid + 1; else hi = mid;
        }
        rs[v] = (uint64_t)lo;
    }
}

__global__ void kp_slice_rs(int64_t nloc, const int64_t *grs, int64_t lo, uint64_t *rs) {
    PSTRIDE(v, nloc + 1) rs[v] = (uint64_t)(grs[lo + v] - grs[lo]);
}

__global__ void kp_init(int64_t nloc, int64_t W, int64_t lo, uint32_t root, uint32_t *parent,
                        int32_t *level, uint32_t *F, uint32_t *V) {
    PSTRIDE(i, nloc) {
        const bool r = lo + i == (int64_t)root;
        parent[i] = r ? root : HBFS_NIL;
        level[i] = r ? 0 : -1;
    }
    PSTRIDE(w, W) {
        const uint32_t b = (w == (int64_t)(root >> 5)) ? (1u << (root & 31)) : 0u;
        F[w] = b;
        V[w] = b;
    }
}

// Owned frontier queue from the replicated F.  Rows of >= kSegArcs arcs are
// also cut into segments of kSegArcs arcs (one entry per segment), so a hub
// row spreads over many CTAs instead of serialising one.
constexpr int64_t kSegArcs = 4096;

__global__ void kp_queue(int64_t wloc, int64_t lo, const uint32_t *F, const uint64_t *rs, uint32_t *q,
                         unsigned long long *qn, uint32_t *seg_u, uint64_t *seg_k,
                         unsigned long long *segn) {
    PSTRIDE(j, wloc) {
        uint32_t bits = F[(lo >> 5) + j];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const uint32_t ul = (uint32_t)(j * 32 + b);  // local id
            q[atomicAdd(qn, 1ull)] = ul;
            const uint64_t s = rs[ul], e = rs[ul + 1];
            if (e - s >= 1024) {
                const unsigned long long ns = (e - s + kSegArcs - 1) / kSegArcs;
                const unsigned long long at = atomicAdd(segn, ns);
                for (unsigned long long t = 0; t < ns; ++t) {
                    seg_u[at + t] = ul;
                    seg_k[at + t] = s + t * kSegArcs;
                }
            }
        }
    }
}

// Column blocking of the long-row segments: a segment's targets are sorted, so
// it splits into pieces by target range (2^kRangeBits vertices, 16 MB of
// cand); pieces are ordered by range, so the CTAs working at any moment update
// one or two L2-resident slices of cand/touch instead of the whole array.
constexpr int kRangeBits = 22;

__device__ __forceinline__ void seg_bounds(const uint32_t *seg_u, const uint64_t *seg_k, const uint64_t *rs,
                                           int64_t g, uint32_t &ul, uint64_t &k0, uint64_t &k1) {
    ul = seg_u[g];
    k0 = seg_k[g];
    const uint64_t e = rs[ul + 1];
    k1 = k0 + kSegArcs < e ? k0 + kSegArcs : e;
}

__global__ void kp_pieces_count(const unsigned long long *segn_p, const uint32_t *seg_u, const uint64_t *seg_k,
                                const uint64_t *rs, const uint32_t *adj, unsigned long long *rcnt) {
    const int64_t segn = (int64_t)*segn_p;
    PSTRIDE(g, segn) {
        uint32_t ul;
        uint64_t k0, k1;
        seg_bounds(seg_u, seg_k, rs, g, ul, k0, k1);
        const uint32_t rf = adj[k0] >> kRangeBits, rl = adj[k1 - 1] >> kRangeBits;
        for (uint32_t r = rf; r <= rl; ++r) atomicAdd(&rcnt[r], 1ull);
    }
}

// rcnt[0..R) -> exclusive offsets in rcur[0..R), total in rcur[R]
__global__ void kp_pieces_scan(int R, const unsigned long long *rcnt, unsigned long long *rcur) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long run = 0;
        for (int r = 0; r < R; ++r) {
            rcur[r] = run;
            run += rcnt[r];
        }
        rcur[R] = run;
    }
}

struct Piece {
    uint64_t a0, a1;  // arc range of the piece
    uint32_t u, pad;  // local row
};

// warp per segment, lane per range: the piece bounds are found here (many
// independent binary searches in flight) rather than by the expanding CTA
__global__ void kp_pieces_fill(const unsigned long long *segn_p, const uint32_t *seg_u, const uint64_t *seg_k,
                               const uint64_t *rs, const uint32_t *adj, unsigned long long *rcur,
                               Piece *pieces) {
    const int64_t segn = (int64_t)*segn_p;
    const int lane = threadIdx.x & 31;
    for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < segn;
         g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        uint32_t ul;
        uint64_t k0, k1;
        seg_bounds(seg_u, seg_k, rs, g, ul, k0, k1);
        const uint32_t rf = adj[k0] >> kRangeBits, rl = adj[k1 - 1] >> kRangeBits;
        for (uint32_t r = rf + lane; r <= rl; r += 32) {
            uint64_t b[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {  // lower_bound of the range edges in the sorted segment
                const uint64_t x = (uint64_t)(r + t) << kRangeBits;
                uint64_t a = k0, c = k1;
                while (a < c) {
                    const uint64_t mid = (a + c) >> 1;
                    if ((uint64_t)adj[mid] < x) a = mid + 1; else c = mid;
                }
                b[t] = a;
            }
            pieces[atomicAdd(&rcur[r], 1ull)] = Piece{b[0], b[1], ul, 0u};
        }
    }
}

// Top-down expansion.  Every arc into an unvisited target lowers cand[v]
// (atomicMin) and marks v in the touch bitmap (a reduction, no return): both
// fire-and-forget.  The records are built afterwards by a scan of the touch
// bitmap in vertex order, which is owner order (owner blocks are contiguous
// word ranges), so no per-target append and no shared counter.
__device__ __forceinline__ void td_arc(uint32_t v, int32_t u, const uint32_t *V, int32_t *cand,
                                       uint32_t *touch) {
    const uint32_t b = 1u << (v & 31);
    if (V[v >> 5] & b) return;
    atomicMin(&cand[v], u);
    if (!(__ldcg(&touch[v >> 5]) & b)) atomicOr(&touch[v >> 5], b);
}

// Short rows (< 1024 arcs): warp per row; long rows: CTA per kSegArcs-arc
// segment.  Counts are read on the device (no host round trip per layer).
__global__ void kp_td(const uint32_t *q, const unsigned long long *qn_p, int64_t lo, const uint64_t *rs,
                      const uint32_t *adj, const uint32_t *V, int32_t *cand, uint32_t *touch,
                      const uint32_t *seg_u, const uint64_t *seg_k, const unsigned long long *segn_p,
                      const Piece *pieces, const unsigned long long *pieces_n_p) {
    const int lane = threadIdx.x & 31;
    const int64_t qn = (int64_t)*qn_p, segn = (int64_t)*segn_p;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < qn;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t ul = q[i];
        const uint64_t s = rs[ul], e = rs[ul + 1];
        if (e - s >= 1024) continue;
        const int32_t u = (int32_t)(lo + ul);
        for (uint64_t k = s + lane; k < e; k += 32) td_arc(adj[k], u, V, cand, touch);
    }
    (void)segn;
    // long-row pieces in range order, CTA per piece, 4 arcs per thread per step
    // (loads of all four issued before their tests)
    const int64_t npieces = (int64_t)pieces_n_p[0];
    for (int64_t i = blockIdx.x; i < npieces; i += gridDim.x) {
        const Piece pc = pieces[i];
        const int32_t u = (int32_t)(lo + pc.u);
        for (uint64_t kb = pc.a0; kb < pc.a1; kb += 4 * (uint64_t)blockDim.x) {
            uint32_t v[4];
            bool ok[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint64_t k = kb + threadIdx.x + (uint64_t)j * blockDim.x;
                ok[j] = k < pc.a1;
                v[j] = ok[j] ? adj[k] : 0u;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (ok[j]) td_arc(v[j], u, V, cand, touch);
        }
    }
    (void)segn;
    (void)seg_u;
    (void)seg_k;
}

__global__ void kp_touch_popc(int64_t W, const uint32_t *touch, uint32_t *cnt) {
    PSTRIDE(w, W) cnt[w] = __popc(touch[w]);
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[W] = 0;
}

// Records per owner o = touched vertices in its word block [o*wper, (o+1)*wper).
__global__ void kp_owner_counts(int world, int64_t wper, int64_t W, const uint32_t *excl, int64_t *counts) {
    const int o = threadIdx.x;
    if (o < world) {
        const int64_t a = o * wper < W ? o * wper : W, b = (o + 1) * wper < W ? (o + 1) * wper : W;
        counts[o] = (int64_t)excl[b] - (int64_t)excl[a];
    }
}

// Records (parent << 32 | v) in vertex order = owner order, at the scanned
// word offsets; resets cand and touch behind itself.
__global__ void kp_td_pack(int64_t W, const uint32_t *excl, int32_t *cand, uint32_t *touch,
                           unsigned long long *rec) {
    PSTRIDE(w, W) {
        uint32_t bits = touch[w];
        if (!bits) continue;
        touch[w] = 0u;
        unsigned long long pos = excl[w];
        for (; bits; bits &= bits - 1) {
            const uint32_t v = (uint32_t)(w * 32 + __ffs(bits) - 1);
            rec[pos++] = ((unsigned long long)(uint32_t)cand[v] << 32) | v;
            cand[v] = 0x7FFFFFFF;
        }
    }
}

// Owner side, pass 1: MIN over every rank's record for the same vertex.
__global__ void kp_td_recv_min(const unsigned long long *rec, int64_t nrec, int64_t lo,
                               int32_t *candown) {
    PSTRIDE(k, nrec) {
        const unsigned long long r = rec[k];
        atomicMin(&candown[(int64_t)(uint32_t)r - lo], (int32_t)(r >> 32));
    }
}

// Owner side, pass 2: the first record of each vertex claims it (next-slice
// bit), writes parent/level from the reduced candidate and resets it.
__global__ void kp_td_recv_claim(const unsigned long long *rec, int64_t nrec, int64_t lo,
                                 int32_t depth1, const uint64_t *rs, int32_t *candown,
                                 uint32_t *parent, int32_t *level, uint32_t *next,
                                 unsigned long long *ctr) {
    unsigned long long c_cnt = 0, c_deg = 0;
    PSTRIDE(k, nrec) {
        const int64_t lv = (int64_t)(uint32_t)rec[k] - lo;
        const uint32_t b = 1u << (lv & 31);
        if (atomicOr(&next[lv >> 5], b) & b) continue;
        parent[lv] = (uint32_t)candown[lv];
        level[lv] = depth1;
        candown[lv] = 0x7FFFFFFF;
        c_cnt += 1;
        c_deg += (unsigned long long)(rs[lv + 1] - rs[lv]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        c_cnt += __shfl_down_sync(0xffffffffu, c_cnt, o);
        c_deg += __shfl_down_sync(0xffffffffu, c_deg, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (c_cnt) atomicAdd(&ctr[0], c_cnt);
        if (c_deg) atomicAdd(&ctr[1], c_deg);
    }
}

// Records applied to the persistent kernel's state: every record lowers the
// owned parent (NIL-initialised; the rank's own arcs did the same in the
// kernel); the first claim of the next-frontier bit stamps the level and
// counts the vertex.
__global__ void kp_apply_persist(const unsigned long long *rec, int64_t nrec, int64_t lo, int32_t depth1,
                                 const uint64_t *rs, uint32_t *parent, int32_t *level, uint32_t *out_plane,
                                 unsigned long long *cnt) {
    unsigned long long c_cnt = 0, c_deg = 0;
    PSTRIDE(k, nrec) {
        const unsigned long long r = rec[k];
        const uint32_t v = (uint32_t)r;
        const int64_t lv = (int64_t)v - lo;
        atomicMin(&parent[lv], (uint32_t)(r >> 32));
        const uint32_t b = 1u << (v & 31);
        if (atomicOr(&out_plane[v >> 5], b) & b) continue;
        level[lv] = depth1;
        c_cnt += 1;
        c_deg += (unsigned long long)(rs[lv + 1] - rs[lv]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        c_cnt += __shfl_down_sync(0xffffffffu, c_cnt, o);
        c_deg += __shfl_down_sync(0xffffffffu, c_deg, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (c_cnt) atomicAdd(&cnt[0], c_cnt);
        if (c_deg) atomicAdd(&cnt[1], c_deg);
    }
}


__global__ void kp_fill_i32(int32_t *p, int64_t n, int32_t x) {
    PSTRIDE(i, n) p[i] = x;
}

__global__ void kp_absorb(int64_t W, const uint32_t *next, uint32_t *F, uint32_t *V) {
    PSTRIDE(w, W) {
        const uint32_t x = next[w];
        F[w] = x;
        if (x) V[w] |= x;
    }
}

__global__ void kp_posw(int64_t nloc, int64_t wloc, const uint64_t *rs, uint32_t *posw) {
    PSTRIDE(w, wloc) {
        uint32_t b = 0;
        for (int j = 0; j < 32; ++j) {
            const int64_t v = w * 32 + j;
            if (v < nloc && rs[v + 1] > rs[v]) b |= 1u << j;
        }
        posw[w] = b;
    }
}

static int part_alloc_state(Part *P) {
    HB_CHECK(P->F.alloc(P->W * 4 + 16));
    HB_CHECK(P->V.alloc(P->W * 4 + 16));
    HB_CHECK(P->parent.alloc(P->nloc * 4 + 16));
    HB_CHECK(P->level.alloc(P->nloc * 4 + 16));
    HB_CHECK(P->q.alloc(P->nloc * 4 + 16));
    HB_CHECK(P->scratch.alloc(64));
    HB_CHECK(P->posw.alloc(P->wloc * 4 + 16));
    HB_CHECK(P->bu_scratch.alloc(part_bu_scratch_bytes()));
    HB_CUDA(cudaDeviceSynchronize());  // rs was built on the caller's stream
    kp_posw<<<pgrid(P->wloc), 256>>>(P->nloc, P->wloc, P->rs.as<uint64_t>(), P->posw.as<uint32_t>());
    HB_CHECK(build_heads(P->nloc, P->rs.p, 1, P->adj.as<uint32_t>(), P->posw.as<uint32_t>(), P->pre, P->hd, 0, &P->n_pos));
    {
        const int64_t nseg = P->arcs / kSegArcs + P->nloc / 1024 + 16;
        HB_CHECK(P->seg_u.alloc(nseg * 4));
        HB_CHECK(P->seg_k.alloc(nseg * 8));
        P->nseg_cap = nseg;
        P->ranges = (int)std::max<int64_t>(1, (P->n + (int64_t(1) << kRangeBits) - 1) >> kRangeBits);
        // a segment splits into at most min(ranges, kSegArcs) pieces
        HB_CHECK(P->pieces.alloc(nseg * std::min<int64_t>(P->ranges, kSegArcs) * sizeof(Piece) + 16));
        HB_CHECK(P->rcnt.alloc((2 * P->ranges + 2) * 8));
    }
    HB_CHECK(P->cand.alloc(P->n * 4 + 16));
    HB_CHECK(P->touch.alloc(P->W * 4 + 16));
    HB_CHECK(P->wcnt.alloc((P->W + 1) * 4 + 16));
    HB_CHECK(P->wexcl.alloc((P->W + 1) * 4 + 16));
    P->scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, P->scan_bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (int)(P->W + 1));
    HB_CHECK(P->scan_tmp.alloc(P->scan_bytes + 16));
    HB_CHECK(P->candown.alloc(P->nloc * 4 + 16));
    kp_fill_i32<<<pgrid(P->n), 256>>>(P->cand.as<int32_t>(), P->n, 0x7FFFFFFF);
    kp_fill_i32<<<pgrid(P->nloc), 256>>>(P->candown.as<int32_t>(), P->nloc, 0x7FFFFFFF);
    HB_CUDA(cudaMemset(P->touch.p, 0, P->W * 4));
    HB_CUDA(cudaDeviceSynchronize());
    return HBFS_OK;
}

static int check_range(int64_t n, int64_t lo, int64_t hi) {
    if (lo < 0 || hi > n || lo >= hi || (lo & 31) || ((hi & 31) && hi != n))
        return set_error(HBFS_EINVAL, "owned range must be word aligned inside [0, n)");
    return HBFS_OK;
}

}  // namespace hbfs

using namespace hbfs;

struct hbfs_part : Part {};

extern "C" int hbfs_part_build(const uint32_t *u, const uint32_t *v, int64_t m, int64_t n,
                               int64_t lo, int64_t hi, int dedup, int on_device, void *stream,
                               hbfs_part **out) {
    HB_ENTRY_BEGIN
    clear_error();
    if (!out || m < 0 || n <= 0) return set_error(HBFS_EINVAL, "bad arguments");
    HB_CHECK(check_range(n, lo, hi));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    DevBuf du, dv, k0, k1, tmp, cnt;
    const uint32_t *pu = u, *pv = v;
    if (!on_device) {
        HB_CHECK(du.alloc(m * 4 + 16));
        HB_CHECK(dv.alloc(m * 4 + 16));
        HB_CUDA(cudaMemcpyAsync(du.p, u, m * 4, cudaMemcpyHostToDevice, st));
        HB_CUDA(cudaMemcpyAsync(dv.p, v, m * 4, cudaMemcpyHostToDevice, st));
        pu = du.as<uint32_t>();
        pv = dv.as<uint32_t>();
    }
    int sb = 1;
    while ((int64_t(1) << sb) < n) ++sb;
    HB_CHECK(cnt.alloc(8));
    HB_CUDA(cudaMemsetAsync(cnt.p, 0, 8, st));
    // count first so the key buffer is sized exactly, then fill
    kp_arc_keys<<<pgrid(m), 256, 0, st>>>(m, sb, lo, hi, pu, pv, nullptr, cnt.as<unsigned long long>());
    HB_CUDA(cudaGetLastError());
    unsigned long long kk = 0;
    HB_CUDA(cudaMemcpyAsync(&kk, cnt.p, 8, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    int64_t k = (int64_t)kk;
    HB_CHECK(k0.alloc(k * 8 + 16));
    HB_CUDA(cudaMemsetAsync(cnt.p, 0, 8, st));
    kp_arc_keys<<<pgrid(m), 256, 0, st>>>(m, sb, lo, hi, pu, pv, k0.as<uint64_t>(),
                                          cnt.as<unsigned long long>());
    HB_CUDA(cudaGetLastError());
    hbfs_part *P = new hbfs_part();
    P->n = n;
    P->lo = lo;
    P->hi = hi;
    P->nloc = hi - lo;
    P->W = (n + 31) / 32;
    P->wlo = lo >> 5;
    P->wloc = (P->nloc + 31) / 32;
    P->m_edges = m;
    int rc = HBFS_OK;
    if (!rc) rc = k1.alloc(k * 8 + 16);
    const int key_bits = 2 * sb;
    if (!rc && k > 0) {
        cub::DoubleBuffer<uint64_t> db(k0.as<uint64_t>(), k1.as<uint64_t>());
        size_t tb = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb, db, k, 0, key_bits, st);
        rc = tmp.alloc(tb);
        if (!rc && cub::DeviceRadixSort::SortKeys(tmp.p, tb, db, k, 0, key_bits, st) != cudaSuccess)
            rc = set_error(HBFS_ECUDA, "sort failed");
        uint64_t *sorted = db.Current();
        if (!rc && dedup) {
            DevBuf flags, nsel, tmp2;
            rc = flags.alloc(k);
            if (!rc) rc = nsel.alloc(8);
            if (!rc) {
                kp_dedup_flags<<<pgrid(k), 256, 0, st>>>(k, sb, lo, sorted, flags.as<uint8_t>());
                size_t tb2 = 0;
                cub::DeviceSelect::Flagged(nullptr, tb2, sorted, flags.as<uint8_t>(), db.Alternate(),
                                           nsel.as<int64_t>(), k, st);
                rc = tmp2.alloc(tb2);
                if (!rc) cub::DeviceSelect::Flagged(tmp2.p, tb2, sorted, flags.as<uint8_t>(),
                                                    db.Alternate(), nsel.as<int64_t>(), k, st);
                int64_t h = 0;
                cudaMemcpyAsync(&h, nsel.p, 8, cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                k = h;
                sorted = db.Alternate();
            }
        }
        if (!rc) rc = P->adj.alloc((k + 8) * 4);
        if (!rc) rc = P->rs.alloc((P->nloc + 1) * 8);
        if (!rc) {
            kp_adj<<<pgrid(k), 256, 0, st>>>(k, sb, sorted, P->adj.as<uint32_t>());
            kp_rs<<<pgrid(P->nloc + 1), 256, 0, st>>>(P->nloc, k, sb, sorted, P->rs.as<uint64_t>());
            if (cudaGetLastError() != cudaSuccess) rc = set_error(HBFS_ECUDA, "csr kernels failed");
        }
    } else if (!rc) {
        rc = P->adj.alloc(64);
        if (!rc) rc = P->rs.alloc((P->nloc + 1) * 8);
        if (!rc) cudaMemsetAsync(P->rs.p, 0, (P->nloc + 1) * 8, st);
    }
    P->arcs = k;
    if (!rc) rc = part_alloc_state(P);
    if (!rc && cudaStreamSynchronize(st) != cudaSuccess) rc = set_error(HBFS_ECUDA, "build failed");
    if (rc) {
        delete P;
        return rc;
    }
    *out = P;
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_part_from_csr(const int64_t *row_starts, const uint32_t *adjacency, int64_t n,
                                  int64_t lo, int64_t hi, int64_t m_edges, void *stream,
                                  hbfs_part **out) {
    HB_ENTRY_BEGIN
    clear_error();
    if (!out || !row_starts || n <= 0) return set_error(HBFS_EINVAL, "bad arguments");
    HB_CHECK(check_range(n, lo, hi));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    hbfs_part *P = new hbfs_part();
    P->n = n;
    P->lo = lo;
    P->hi = hi;
    P->nloc = hi - lo;
    P->W = (n + 31) / 32;
    P->wlo = lo >> 5;
    P->wloc = (P->nloc + 31) / 32;
    P->m_edges = m_edges;
    const int64_t a0 = row_starts[lo], a1 = row_starts[hi];
    P->arcs = a1 - a0;
    DevBuf grs;
    int rc = grs.alloc((P->nloc + 1) * 8);
    if (!rc) rc = P->rs.alloc((P->nloc + 1) * 8);
    if (!rc) rc = P->adj.alloc((P->arcs + 8) * 4);
    if (!rc && cudaMemcpyAsync(grs.p, row_starts + lo, (P->nloc + 1) * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
        rc = set_error(HBFS_ECUDA, "copy failed");
    if (!rc && P->arcs > 0 &&
        cudaMemcpyAsync(P->adj.p, adjacency + a0, P->arcs * 4, cudaMemcpyHostToDevice, st) != cudaSuccess)
        rc = set_error(HBFS_ECUDA, "copy failed");
    if (!rc) {
        kp_slice_rs<<<pgrid(P->nloc + 1), 256, 0, st>>>(P->nloc, grs.as<int64_t>(), 0, P->rs.as<uint64_t>());
        if (cudaGetLastError() != cudaSuccess) rc = set_error(HBFS_ECUDA, "slice failed");
    }
    if (!rc) rc = part_alloc_state(P);
    if (!rc && cudaStreamSynchronize(st) != cudaSuccess) rc = set_error(HBFS_ECUDA, "import failed");
    if (rc) {
        delete P;
        return rc;
    }
    *out = P;
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_part_info(const hbfs_part *P, int64_t *n, int64_t *lo, int64_t *hi,
                              int64_t *local_arcs, int64_t *m_edges) {
    if (!P) return set_error(HBFS_EINVAL, "null part");
    if (n) *n = P->n;
    if (lo) *lo = P->lo;
    if (hi) *hi = P->hi;
    if (local_arcs) *local_arcs = P->arcs;
    if (m_edges) *m_edges = P->m_edges;
    return HBFS_OK;
}

extern "C" int hbfs_part_free(hbfs_part *P) {
    HB_ENTRY_BEGIN
    delete P;
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_part_degree(const hbfs_part *P, int64_t v, int64_t *deg) {
    HB_ENTRY_BEGIN
    if (!P || !deg) return set_error(HBFS_EINVAL, "bad arguments");
    *deg = 0;
    if (v < P->lo || v >= P->hi) return HBFS_OK;
    uint64_t h[2];
    HB_CUDA(cudaMemcpy(h, P->rs.as<uint64_t>() + (v - P->lo), 16, cudaMemcpyDeviceToHost));
    *deg = (int64_t)(h[1] - h[0]);
    return HBFS_OK;
    HB_ENTRY_END
}

__global__ void kp_degrees(int64_t count, const uint32_t *ids, int64_t lo, int64_t hi, const uint64_t *rs,
                           int64_t *deg) {
    PSTRIDE(i, count) {
        const int64_t v = ids[i];
        deg[i] = v >= lo && v < hi ? (int64_t)(rs[v - lo + 1] - rs[v - lo]) : 0;
    }
}

// deg[i] = degree of ids[i] if this rank owns it, else 0 (host arrays): summed
// over the ranks these are the global degrees of a candidate list.
extern "C" int hbfs_part_degrees(const hbfs_part *P, const uint32_t *ids, int64_t count, int64_t *deg) {
    HB_ENTRY_BEGIN
    if (!P || !ids || !deg || count < 0) return set_error(HBFS_EINVAL, "bad arguments");
    if (count == 0) return HBFS_OK;
    DevBuf di, dd;
    HB_CHECK(di.alloc(count * 4));
    HB_CHECK(dd.alloc(count * 8));
    HB_CUDA(cudaMemcpy(di.p, ids, count * 4, cudaMemcpyHostToDevice));
    kp_degrees<<<pgrid(count), 256>>>(count, di.as<uint32_t>(), P->lo, P->hi, P->rs.as<uint64_t>(), dd.as<int64_t>());
    HB_CUDA(cudaGetLastError());
    HB_CUDA(cudaMemcpy(deg, dd.p, count * 8, cudaMemcpyDeviceToHost));
    return HBFS_OK;
    HB_ENTRY_END
}

// Exchange volume of the last hbfs_mg_bfs / hbfs_mgl_bfs traversal of this
// part: out[0] records sent (8 bytes each), out[1] records received, out[2]
// layers (one next-frontier all-gather and one counter all-reduce each),
// out[3] top-down record exchanges.
extern "C" int hbfs_part_exchange_stats(const hbfs_part *P, int64_t *out) {
    HB_ENTRY_BEGIN
    if (!P || !out) return set_error(HBFS_EINVAL, "bad arguments");
    for (int k = 0; k < 4; ++k) out[k] = P->stat[k];
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_part_init(hbfs_part *P, int64_t root, void *stream) {
    HB_ENTRY_BEGIN
    if (!P) return set_error(HBFS_EINVAL, "null part");
    if (root < 0 || root >= P->n) return set_error(HBFS_ERANGE, "source out of range");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    kp_init<<<pgrid(std::max(P->nloc, P->W)), 256, 0, st>>>(
        P->nloc, P->W, P->lo, (uint32_t)root, P->parent.as<uint32_t>(), P->level.as<int32_t>(),
        P->F.as<uint32_t>(), P->V.as<uint32_t>());
    HB_CUDA(cudaGetLastError());
    return HBFS_OK;
    HB_ENTRY_END
}

// counters: device uint64[4] = {found, degree sum of found, gathers, fallbacks}
extern "C" int hbfs_part_bu(hbfs_part *P, int32_t depth, int32_t max_pos, uint32_t *next_slice,
                            unsigned long long *counters, void *stream) {
    HB_ENTRY_BEGIN
    if (!P || !next_slice || !counters) return set_error(HBFS_EINVAL, "bad arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the persistent kernel's bottom-up tiles on the owned words (bfs.cu)
    HB_CHECK(part_bu_launch(P->rs.as<uint64_t>(), P->adj.as<uint32_t>(), P->posw.as<uint32_t>(), P->hd.as<uint4>(), P->n_pos, P->pre.as<uint32_t>(), P->n, P->lo,
                            P->nloc, P->arcs, P->F.as<uint32_t>(), P->V.as<uint32_t>(), P->parent.as<uint32_t>(),
                            P->level.as<int32_t>(), next_slice, depth, max_pos, P->fhint, counters,
                            P->bu_scratch.p, st));
    return HBFS_OK;
    HB_ENTRY_END
}

// Global frontier size of the coming bottom-up layer (selects the tiny-frontier
// probe variant, as on one GPU); optional.
extern "C" int hbfs_part_hint_frontier(hbfs_part *P, int64_t v_f) {
    if (!P) return set_error(HBFS_EINVAL, "null part");
    P->fhint = v_f;
    return HBFS_OK;
}

// Records per owner from the touch bitmap (popcount + scan in vertex order).
static int td_owner_counts(Part *P, int world, int64_t wper, int64_t *send_counts, cudaStream_t st) {
    uint32_t *cnt = P->wcnt.as<uint32_t>();
    kp_touch_popc<<<pgrid(P->W + 1), 256, 0, st>>>(P->W, P->touch.as<uint32_t>(), cnt);
    size_t tb = P->scan_bytes;
    HB_CUDA(cub::DeviceScan::ExclusiveSum(P->scan_tmp.p, tb, cnt, P->wexcl.as<uint32_t>(), (int)(P->W + 1), st));
    kp_owner_counts<<<1, 32, 0, st>>>(world, wper, P->W, P->wexcl.as<uint32_t>(), send_counts);
    HB_CUDA(cudaGetLastError());
    return HBFS_OK;
}

// Top-down expansion of the owned frontier for a `world`-rank partition (owner
// blocks of `span` = partition() words * 32 vertices).  send_counts: device
// int64[world], records queued per owner.
extern "C" int hbfs_part_td_expand(hbfs_part *P, int32_t world, int64_t *send_counts, void *stream) {
    HB_ENTRY_BEGIN
    if (!P || !send_counts || world < 1) return set_error(HBFS_EINVAL, "bad arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t wper = (P->W + world - 1) / world;
    const int64_t span = wper * 32;
    if (P->world != world) {
        P->world = world;
        P->span = span;
    }
    unsigned long long *qn = P->scratch.as<unsigned long long>();  // [0] queue, [1] segments
    HB_CUDA(cudaMemsetAsync(qn, 0, 16, st));
    kp_queue<<<pgrid(P->wloc), 256, 0, st>>>(P->wloc, P->lo, P->F.as<uint32_t>(), P->rs.as<uint64_t>(),
                                             P->q.as<uint32_t>(), qn, P->seg_u.as<uint32_t>(),
                                             P->seg_k.as<uint64_t>(), qn + 1);
    unsigned long long *rcnt = P->rcnt.as<unsigned long long>(), *rcur = rcnt + P->ranges;
    HB_CUDA(cudaMemsetAsync(rcnt, 0, P->ranges * 8, st));
    kp_pieces_count<<<pgrid(P->nseg_cap), 256, 0, st>>>(qn + 1, P->seg_u.as<uint32_t>(), P->seg_k.as<uint64_t>(),
                                                       P->rs.as<uint64_t>(), P->adj.as<uint32_t>(), rcnt);
    kp_pieces_scan<<<1, 32, 0, st>>>(P->ranges, rcnt, rcur);
    kp_pieces_fill<<<pgrid(P->nseg_cap * 32), 256, 0, st>>>(qn + 1, P->seg_u.as<uint32_t>(), P->seg_k.as<uint64_t>(),
                                                           P->rs.as<uint64_t>(), P->adj.as<uint32_t>(), rcur,
                                                           P->pieces.as<Piece>());
    kp_td<<<148 * 8, 256, 0, st>>>(P->q.as<uint32_t>(), qn, P->lo, P->rs.as<uint64_t>(), P->adj.as<uint32_t>(),
                                   P->V.as<uint32_t>(), P->cand.as<int32_t>(), P->touch.as<uint32_t>(),
                                   P->seg_u.as<uint32_t>(), P->seg_k.as<uint64_t>(), qn + 1,
                                   P->pieces.as<Piece>(), rcur + P->ranges);
    HB_CHECK(td_owner_counts(P, world, wper, send_counts, st));
    return HBFS_OK;
    HB_ENTRY_END
}

// records: device uint64[sum(send_counts)], packed by owner; resets the
// expansion state for the next layer.
extern "C" int hbfs_part_td_pack(hbfs_part *P, uint64_t *records, void *stream) {
    HB_ENTRY_BEGIN
    if (!P || !records || P->world < 1) return set_error(HBFS_EINVAL, "bad arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    kp_td_pack<<<pgrid(P->W), 256, 0, st>>>(P->W, P->wexcl.as<uint32_t>(), P->cand.as<int32_t>(),
                                            P->touch.as<uint32_t>(),
                                            reinterpret_cast<unsigned long long *>(records));
    HB_CUDA(cudaGetLastError());
    return HBFS_OK;
    HB_ENTRY_END
}

// records: device uint64[nrec] received from every rank (vertices owned here).
extern "C" int hbfs_part_td_apply(hbfs_part *P, int32_t depth, const uint64_t *records,
                                  int64_t nrec, uint32_t *next_slice,
                                  unsigned long long *counters, void *stream) {
    HB_ENTRY_BEGIN
    if (!P || (!records && nrec) || nrec < 0 || !next_slice || !counters)
        return set_error(HBFS_EINVAL, "bad arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    HB_CUDA(cudaMemsetAsync(counters, 0, 32, st));
    if (nrec > 0) {
        const unsigned long long *r = reinterpret_cast<const unsigned long long *>(records);
        kp_td_recv_min<<<pgrid(nrec), 256, 0, st>>>(r, nrec, P->lo, P->candown.as<int32_t>());
        kp_td_recv_claim<<<pgrid(nrec), 256, 0, st>>>(r, nrec, P->lo, depth + 1, P->rs.as<uint64_t>(),
                                                      P->candown.as<int32_t>(), P->parent.as<uint32_t>(),
                                                      P->level.as<int32_t>(), next_slice, counters);
        HB_CUDA(cudaGetLastError());
    }
    return HBFS_OK;
    HB_ENTRY_END
}

// next_full: device uint32[W] (all-gathered next frontier): F = next, V |= next
extern "C" int hbfs_part_absorb(hbfs_part *P, const uint32_t *next_full, void *stream) {
    HB_ENTRY_BEGIN
    if (!P || !next_full) return set_error(HBFS_EINVAL, "bad arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    kp_absorb<<<pgrid(P->W), 256, 0, st>>>(P->W, next_full, P->F.as<uint32_t>(), P->V.as<uint32_t>());
    HB_CUDA(cudaGetLastError());
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_part_outputs(hbfs_part *P, uint32_t *parent, int32_t *level, int on_device,
                                 void *stream) {
    HB_ENTRY_BEGIN
    if (!P) return set_error(HBFS_EINVAL, "null part");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (parent) HB_CUDA(cudaMemcpyAsync(parent, P->parent.p, P->nloc * 4, k, st));
    if (level) HB_CUDA(cudaMemcpyAsync(level, P->level.p, P->nloc * 4, k, st));
    HB_CUDA(cudaStreamSynchronize(st));
    return HBFS_OK;
    HB_ENTRY_END
}

// ------------------------------------------------------------------------
// Multi-GPU traversal loop in C++ over NCCL: one process per GPU, the same
// per-layer steps as mgpu.DistBfs (which keeps the host logic testable with
// gloo on CPU) without Python in the loop.  Per layer: the rank's kernels,
// in-place ncclAllGather of the next-frontier slices, ncclAllReduce of the
// four counters, and on top-down layers grouped ncclSend/ncclRecv for the
// per-owner counts and the 8-byte records.  Host round trips per layer: the
// counter read for the direction decision (hybrid.py:123-173) and, on
// top-down layers, the record counts (NCCL needs split sizes on the host).
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <vector>

// NCCL is resolved at first use (dlopen by SONAME), not linked: the process
// may already hold torch's libnccl.so.2, and a second, older copy loaded first
// by this library would shadow the symbols torch needs.  Python callers import
// torch (and let it load its NCCL) before the first multi-GPU call.
namespace {
struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclGetErrorString) getErrorString = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    bool ok = false;
};

const NcclApi &nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
#define HB_SYM(field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, #name))
        HB_SYM(getUniqueId, ncclGetUniqueId);
        HB_SYM(commInitRank, ncclCommInitRank);
        HB_SYM(commDestroy, ncclCommDestroy);
        HB_SYM(getErrorString, ncclGetErrorString);
        HB_SYM(groupStart, ncclGroupStart);
        HB_SYM(groupEnd, ncclGroupEnd);
        HB_SYM(send, ncclSend);
        HB_SYM(recv, ncclRecv);
        HB_SYM(allGather, ncclAllGather);
        HB_SYM(allReduce, ncclAllReduce);
#undef HB_SYM
        a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.getErrorString && a.groupStart &&
               a.groupEnd && a.send && a.recv && a.allGather && a.allReduce;
        return a;
    }();
    return api;
}
}  // namespace

#define HB_NCCL(expr)                                                                       \
    do {                                                                                    \
        ncclResult_t r_ = (expr);                                                           \
        if (r_ != ncclSuccess)                                                              \
            return ::hbfs::set_error(HBFS_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #expr, \
                                     nccl().getErrorString(r_));                            \
    } while (0)
#define HB_NCCL_API()                                                                        \
    do {                                                                                     \
        if (!nccl().ok) return ::hbfs::set_error(HBFS_ENCCL, "libnccl.so.2 not loadable");   \
    } while (0)

struct hbfs_mg {
    ncclComm_t comm = nullptr;
    int world = 0, rank = 0;
    hbfs::DevBuf next_full, ctr, counts, recs_s, recs_r, scal;
    size_t cap_s = 0, cap_r = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    ~hbfs_mg() {
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (comm) nccl().commDestroy(comm);
    }
};

extern "C" int hbfs_nccl_unique_id(void *out, int64_t bytes) {
    HB_ENTRY_BEGIN
    clear_error();
    if (!out || bytes < (int64_t)sizeof(ncclUniqueId)) return set_error(HBFS_EINVAL, "need %d bytes", (int)sizeof(ncclUniqueId));
    HB_NCCL_API();
    ncclUniqueId id;
    HB_NCCL(nccl().getUniqueId(&id));
    memcpy(out, &id, sizeof(id));
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_mg_init(const void *unique_id, int32_t world, int32_t rank, hbfs_mg **out) {
    HB_ENTRY_BEGIN
    clear_error();
    if (!unique_id || !out || world < 1 || rank < 0 || rank >= world) return set_error(HBFS_EINVAL, "bad arguments");
    HB_NCCL_API();
    hbfs_mg *M = new hbfs_mg();
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof(id));
    ncclResult_t r = nccl().commInitRank(&M->comm, world, id, rank);
    if (r != ncclSuccess) {
        M->comm = nullptr;
        delete M;
        return set_error(HBFS_ENCCL, "ncclCommInitRank: %s", nccl().getErrorString(r));
    }
    M->world = world;
    M->rank = rank;
    int rc = M->ctr.alloc(64);
    if (!rc) rc = M->counts.alloc(16 * world + 16);
    if (!rc) rc = M->scal.alloc(64);
    if (!rc && (cudaEventCreate(&M->ev0) != cudaSuccess || cudaEventCreate(&M->ev1) != cudaSuccess))
        rc = set_error(HBFS_ECUDA, "cudaEventCreate failed");
    if (rc) {
        delete M;
        return rc;
    }
    *out = M;
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_mg_free(hbfs_mg *M) {
    HB_ENTRY_BEGIN
    delete M;
    return HBFS_OK;
    HB_ENTRY_END
}

namespace {
int grow(hbfs::DevBuf &b, size_t &cap, size_t need) {
    if (need <= cap) return HBFS_OK;
    size_t c = std::max<size_t>(need + need / 4, 1 << 16);
    HB_CHECK(b.alloc(c * 8));
    cap = c;
    return HBFS_OK;
}
}  // namespace

// The per-layer loop over the persistent partition kernel (bfs.cu
// part_trav_layer).  Either one part per process with NCCL (M != nullptr),
// or all `world` parts of a partition in this process on one device (M ==
// nullptr: exchanges are device copies; used to test P ranks on one GPU).
static int persist_loop(hbfs_part **Ps, int nparts, hbfs_mg *M, int world, int64_t root,
                        const hbfs_params *p, hbfs_layer_row *trace, int64_t trace_cap, int64_t *n_layers,
                        float *device_ms, cudaStream_t st) {
    if (p->parent_mode != HBFS_PARENT_MINID) return set_error(HBFS_EINVAL, "partitions use min-id parents");
    Part *P0 = Ps[0];
    const int64_t n = P0->n, W = P0->W;
    const int64_t wper = (W + world - 1) / world, nw_pad = wper * world;
    for (int i = 0; i < nparts; ++i) {
        Part *P = Ps[i];
        const int rank = M ? M->rank : i;
        if (P->n != n || P->lo != std::min<int64_t>(rank * wper * 32, n))
            return set_error(HBFS_EINVAL, "partition does not match rank/world");
        if (!P->trav) {
            int rc = HBFS_OK;
            P->trav = part_trav_create(n, P->lo, P->nloc, P->arcs, P->rs.as<uint64_t>(), P->adj.as<uint32_t>(),
                                       P->posw.as<uint32_t>(), P->hd.as<uint4>(), P->n_pos, P->pre.as<uint32_t>(), P->parent.as<uint32_t>(),
                                       P->level.as<int32_t>(),
                                       reinterpret_cast<uint32_t *>(P->cand.as<int32_t>()), P->touch.as<uint32_t>(),
                                       &rc, nw_pad);
            if (!P->trav) return rc;
        }
        // record buffers at their bounds (a rank sends at most one record per
        // non-owned vertex and receives at most world-1 per owned vertex, both
        // <= n): growing them inside a traversal costs milliseconds
        if (P->cap_s < (size_t)n + 1) {
            HB_CHECK(P->recs_s.alloc((n + 1) * 8));
            P->cap_s = n + 1;
        }
        if (P->cap_r < (size_t)n + 1) {
            HB_CHECK(P->recs_r.alloc((n + 1) * 8));
            P->cap_r = n + 1;
        }
        if (!P->acnt.p) HB_CHECK(P->acnt.alloc(64));
        if (!P->lay.p) HB_CHECK(P->lay.alloc(64));
        if (!P->h_acnt && cudaMallocHost(&P->h_acnt, 32) != cudaSuccess)
            return set_error(HBFS_ECUDA, "cudaMallocHost failed");
        if (!P->counts_dev.p) HB_CHECK(P->counts_dev.alloc(16 * world + 16));
    }
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    HB_CUDA(cudaEventCreate(&ev0));
    HB_CUDA(cudaEventCreate(&ev1));
    HB_CUDA(cudaEventRecord(ev0, st));
    // root degree and global arc count
    int64_t h2[3] = {0, 0, 0};  // root degree, arcs, vertices with degree > 0
    for (int i = 0; i < nparts; ++i) {
        int64_t d = 0;
        if (root >= Ps[i]->lo && root < Ps[i]->hi) HB_CHECK(hbfs_part_degree(Ps[i], root, &d));
        h2[0] += d;
        h2[1] += Ps[i]->arcs;
        h2[2] += Ps[i]->n_pos;
    }
    if (M && world > 1) {
        int64_t *scal = M->scal.as<int64_t>();
        HB_CUDA(cudaMemcpyAsync(scal, h2, 24, cudaMemcpyHostToDevice, st));
        HB_NCCL(nccl().allReduce(scal, scal, 3, ncclInt64, ncclSum, M->comm, st));
        HB_CUDA(cudaMemcpyAsync(h2, scal, 24, cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaStreamSynchronize(st));
    }
    const int64_t n_pos = h2[2], ratio = bu_exec_ratio();
    Heur H;
    H.heuristic = p->heuristic;
    H.counter_mode = p->counter_mode;
    H.force = p->force_direction;
    H.alpha = p->alpha;
    H.beta = p->beta;
    H.n = n;
    int64_t v_f = 1, e_f = h2[0], eu_v = n - 1, eu_e = h2[1] - h2[0], prev_vf = 0, layer = 0;
    int cur = HBFS_TOP_DOWN;
    std::vector<int64_t> hc((size_t)2 * world * nparts);  // [part][send world | recv world]
    auto t_layer = std::chrono::steady_clock::now();
    for (int i = 0; i < nparts; ++i) Ps[i]->stat[0] = Ps[i]->stat[1] = Ps[i]->stat[2] = Ps[i]->stat[3] = 0;
    while (v_f > 0) {
        int64_t fv, gv;
        const int d = decide(H, cur, v_f, e_f, eu_v, eu_e, prev_vf, &fv, &gv);
        const int64_t state[6] = {layer, v_f, e_f, eu_v, eu_e, prev_vf};
        // The layer's counter totals are summed on the device (this process's
        // parts, then all-reduced over the ranks) and read back with the one
        // stream synchronisation that ends the layer; a top-down layer of a
        // partition with more than one rank needs one more, for the record
        // counts NCCL takes from the host.
        unsigned long long *lay = P0->lay.as<unsigned long long>();
        // records only after a real top-down expansion with remote targets
        const bool exchange = d == HBFS_TOP_DOWN && world > 1 && !bu_executes(d, 1, eu_v, e_f, n, n_pos, ratio);
        // one part in this process and no records to add: the kernel itself
        // leaves the layer totals in `lay`
        const bool direct = nparts == 1 && !exchange;
        if (!direct) HB_CUDA(cudaMemsetAsync(lay, 0, 32, st));
        for (int i = 0; i < nparts; ++i)  // asynchronous
            HB_CHECK(part_trav_layer(Ps[i]->trav, state, cur, layer == 0, (uint32_t)root, p, n_pos,
                                     direct ? lay : nullptr, world == 1, st));
        if (exchange) {
            for (int i = 0; i < nparts; ++i)
                HB_CHECK(td_owner_counts(Ps[i], world, wper, Ps[i]->counts_dev.as<int64_t>(), st));
            if (M) {
                int64_t *sc = Ps[0]->counts_dev.as<int64_t>(), *rc = sc + world;
                HB_NCCL(nccl().groupStart());
                for (int r = 0; r < world; ++r) {
                    HB_NCCL(nccl().send(sc + r, 1, ncclInt64, r, M->comm, st));
                    HB_NCCL(nccl().recv(rc + r, 1, ncclInt64, r, M->comm, st));
                }
                HB_NCCL(nccl().groupEnd());
                HB_CUDA(cudaMemcpyAsync(hc.data(), sc, 16 * world, cudaMemcpyDeviceToHost, st));
            } else {
                for (int i = 0; i < nparts; ++i)
                    HB_CUDA(cudaMemcpyAsync(hc.data() + (size_t)2 * world * i, Ps[i]->counts_dev.p, 8 * world,
                                            cudaMemcpyDeviceToHost, st));
            }
            HB_CUDA(cudaStreamSynchronize(st));
            if (!M)  // recv[i][s] = send[s][i]
                for (int i = 0; i < nparts; ++i)
                    for (int sr = 0; sr < world; ++sr) hc[(size_t)2 * world * i + world + sr] = hc[(size_t)2 * world * sr + i];
            for (int i = 0; i < nparts; ++i) {
                Part *P = Ps[i];
                int64_t ns = 0, nr = 0;
                for (int r = 0; r < world; ++r) {
                    ns += hc[(size_t)2 * world * i + r];
                    nr += hc[(size_t)2 * world * i + world + r];
                }
                P->stat[0] += ns;
                P->stat[1] += nr;
                P->stat[3] += 1;
                if ((size_t)ns + 1 > P->cap_s) {
                    HB_CHECK(P->recs_s.alloc((ns + ns / 4 + 1024) * 8));
                    P->cap_s = ns + ns / 4 + 1024;
                }
                if ((size_t)nr + 1 > P->cap_r) {
                    HB_CHECK(P->recs_r.alloc((nr + nr / 4 + 1024) * 8));
                    P->cap_r = nr + nr / 4 + 1024;
                }
                kp_td_pack<<<pgrid(P->W), 256, 0, st>>>(P->W, P->wexcl.as<uint32_t>(), P->cand.as<int32_t>(),
                                                        P->touch.as<uint32_t>(), P->recs_s.as<unsigned long long>());
                HB_CUDA(cudaGetLastError());
            }
            if (M) {
                const int64_t *h = hc.data();
                HB_NCCL(nccl().groupStart());
                int64_t os = 0, orr = 0;
                for (int r = 0; r < world; ++r) {
                    if (h[r]) HB_NCCL(nccl().send(Ps[0]->recs_s.as<uint64_t>() + os, (size_t)h[r], ncclUint64, r, M->comm, st));
                    if (h[world + r])
                        HB_NCCL(nccl().recv(Ps[0]->recs_r.as<uint64_t>() + orr, (size_t)h[world + r], ncclUint64, r, M->comm, st));
                    os += h[r];
                    orr += h[world + r];
                }
                HB_NCCL(nccl().groupEnd());
            } else {
                for (int i = 0; i < nparts; ++i) {  // receiver i gathers sender segments in rank order
                    int64_t orr = 0;
                    for (int sr = 0; sr < nparts; ++sr) {
                        int64_t os = 0;
                        for (int r = 0; r < i; ++r) os += hc[(size_t)2 * world * sr + r];
                        const int64_t c = hc[(size_t)2 * world * sr + i];
                        if (c)
                            HB_CUDA(cudaMemcpyAsync(Ps[i]->recs_r.as<uint64_t>() + orr, Ps[sr]->recs_s.as<uint64_t>() + os,
                                                    c * 8, cudaMemcpyDeviceToDevice, st));
                        orr += c;
                    }
                }
            }
            for (int i = 0; i < nparts; ++i) {
                Part *P = Ps[i];
                int64_t nr = 0;
                for (int r = 0; r < world; ++r) nr += hc[(size_t)2 * world * i + world + r];
                HB_CUDA(cudaMemsetAsync(P->acnt.p, 0, 16, st));
                if (nr)
                    kp_apply_persist<<<pgrid(nr), 256, 0, st>>>(P->recs_r.as<unsigned long long>(), nr, P->lo,
                                                               (int32_t)layer + 1, P->rs.as<uint64_t>(),
                                                               P->parent.as<uint32_t>(), P->level.as<int32_t>(),
                                                               part_trav_plane(P->trav, layer + 1),
                                                               P->acnt.as<unsigned long long>());
            }
        }
        if (!direct)
            for (int i = 0; i < nparts; ++i)
                HB_CHECK(part_trav_add_counters(Ps[i]->trav, layer,
                                                exchange ? Ps[i]->acnt.as<unsigned long long>() : nullptr, lay, st));
        // next frontier: every rank's owned words of plane layer+1 to everyone
        // (the next launch ORs the all-gathered plane into the visited bitmap)
        if (M && world > 1) {
            uint32_t *pl = part_trav_plane(Ps[0]->trav, layer + 1);
            HB_NCCL(nccl().allGather(pl + M->rank * wper, pl, (size_t)wper, ncclUint32, M->comm, st));
            HB_NCCL(nccl().allReduce(lay, lay, 4, ncclUint64, ncclSum, M->comm, st));
        } else if (!M) {
            for (int i = 0; i < nparts; ++i)
                for (int sr = 0; sr < nparts; ++sr)
                    if (sr != i)
                        HB_CUDA(cudaMemcpyAsync(part_trav_plane(Ps[i]->trav, layer + 1) + sr * wper,
                                                part_trav_plane(Ps[sr]->trav, layer + 1) + sr * wper, wper * 4,
                                                cudaMemcpyDeviceToDevice, st));
        }
        HB_CUDA(cudaMemcpyAsync(P0->h_acnt, lay, 32, cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaStreamSynchronize(st));
        const unsigned long long *tot = P0->h_acnt;
        if (trace && layer < trace_cap) {
            hbfs_layer_row &r = trace[layer];
            r.layer = (int32_t)(layer + 1);
            r.direction = d;
            r.v_f = v_f;
            r.e_f = e_f;
            r.e_u = p->counter_mode ? eu_e : eu_v;
            r.f_value = fv;
            r.g_value = gv;
            r.fallback_count = !p->use_simd || d == HBFS_TOP_DOWN ? 0 : (int64_t)tot[3];
            r.gather_count = !p->use_simd ? 0 : d == HBFS_TOP_DOWN ? e_f : (int64_t)tot[2];
            const auto now = std::chrono::steady_clock::now();
            r.elapsed = std::chrono::duration<double>(now - t_layer).count();  // host wall of the layer
            t_layer = now;
        }
        for (int i = 0; i < nparts; ++i) Ps[i]->stat[2] += 1;
        prev_vf = v_f;
        v_f = (int64_t)tot[0];
        e_f = (int64_t)tot[1];
        eu_v -= v_f;
        eu_e -= e_f;
        cur = d;
        ++layer;
    }
    for (int i = 0; i < nparts; ++i) HB_CHECK(part_trav_levels(Ps[i]->trav, layer, st));
    HB_CUDA(cudaEventRecord(ev1, st));
    HB_CUDA(cudaEventSynchronize(ev1));
    if (device_ms) HB_CUDA(cudaEventElapsedTime(device_ms, ev0, ev1));
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    if (n_layers) *n_layers = layer;
    return HBFS_OK;
}

extern "C" int hbfs_mg_bfs(hbfs_mg *M, hbfs_part *P, int64_t root, const hbfs_params *p,
                           hbfs_layer_row *trace, int64_t trace_cap, int64_t *n_layers,
                           float *device_ms, void *stream) {
    HB_ENTRY_BEGIN
    clear_error();
    if (!M || !P || !p) return set_error(HBFS_EINVAL, "null argument");
    if (root < 0 || root >= P->n)
        return set_error(HBFS_ERANGE, "source %lld out of range [0, %lld)", (long long)root, (long long)P->n);
    hbfs_part *ps[1] = {P};
    return persist_loop(ps, 1, M, M->world, root, p, trace, trace_cap, n_layers, device_ms,
                        static_cast<cudaStream_t>(stream));
    HB_ENTRY_END
}

// All `world` parts of a partition in this process (one device): the same
// loop with device copies for the exchanges (tests P ranks on one GPU).
extern "C" int hbfs_mgl_bfs(hbfs_part **parts, int32_t world, int64_t root, const hbfs_params *p,
                            hbfs_layer_row *trace, int64_t trace_cap, int64_t *n_layers, float *device_ms,
                            void *stream) {
    HB_ENTRY_BEGIN
    clear_error();
    if (!parts || world < 1 || !p) return set_error(HBFS_EINVAL, "bad arguments");
    for (int i = 0; i < world; ++i)
        if (!parts[i]) return set_error(HBFS_EINVAL, "null part");
    if (root < 0 || root >= parts[0]->n)
        return set_error(HBFS_ERANGE, "source %lld out of range [0, %lld)", (long long)root, (long long)parts[0]->n);
    return persist_loop(parts, world, nullptr, world, root, p, trace, trace_cap, n_layers, device_ms,
                        static_cast<cudaStream_t>(stream));
    HB_ENTRY_END
}
