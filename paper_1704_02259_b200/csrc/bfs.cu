// Hybrid (direction-optimising) BFS for sm_100a — one persistent cooperative
// kernel per traversal.
//
// Replaces, as one device-resident loop, the reference's per-layer controller
// hybrid.hybrid_bfs (hybrid.py:83-175), its engine dispatch (engine.py:81-155),
// the native layer kernels top_down_layer / top_down_chunked /
// bottom_up_layer / bottom_up_multiple_set (_native.pyx:65-239, bu_probe.h)
// and the per-layer counters (bfs_scalar.py:18-26).
//
// Layout in HBM (per graph, reused by every root):
//   rs     OffT[n+1]    row starts (uint32 when arcs < 2^32, else uint64)
//   adj    u32[arcs]    sorted rows (csr.py:61-64)
//   posw   u32[W]       deg>0 bitmap (engine.py:29-57 `posw`)
//   hd     uint4[R]     head records {degree, row[0..2]}, rank-packed over the R
//                        vertices with degree > 0; behind them (same slots) the
//                        32-byte second-tier records {row start, row[3..9]}
//   pre    u32[W+1]     head records before bitmap word w
//   parent u32[n], level i32[n]
//   bits   u32[33W]     vis | a ring of kPlanes depth planes — LSB-first bitmaps
//                        (frontier.py:3-6); plane 1 + d % kPlanes holds depth d
//   q/qo/qr             frontier queue: vertex, exclusive degree prefix (arc
//                        offset), row start — double-buffered
//   cs     u32[2*NC]    chunk starts: queue index holding arc c*kTdChunk
//
// Invariants at the start of layer L (frontier = depth L):
//   in  = plane(L) = frontier bitmap; out = plane(L+1) is all-zero;
//   spare = plane(L+2) is cleared during L (its levels stamped first if the ring wrapped)
//   vis | in = every vertex discovered so far (vis may lag by the frontier)
//   queue buffer L%2 valid iff the frontier was produced by the top-down claim
//   path (kind 0); harvest and bottom-up layers leave only the bitmap (kind 1)
// Parents follow the reference's rule: the minimum-id neighbour one
// level up.  Bottom-up layers get it directly (first hit in the sorted row);
// top-down layers take the atomicMin over every arc into a vertex unvisited
// before the layer (parent_mode MINID).  parent_mode ANY lets the first
// claimer win (one visited-bitmap claim per vertex, Graph500-valid trees).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace hbfs {

constexpr int kTdItems = 4;
constexpr int kTdChunk = kBlock * kTdItems;  // arcs per CTA work item
// uint4 row probes per lane before the warp-cooperative scan: 2 normally, 4 in
// bottom-up layers whose frontier is tiny (most rows are scanned to the end)
constexpr int kLaneVecs = 2;
constexpr int kLaneVecsScan = 4;
constexpr int kTdMaxSub = 8;  // top-down chunk split on small layers (2048 / 8 = 256 arcs per CTA)
constexpr uint64_t kTailLong = 256;  // open rows longer than this use the whole-warp scan
constexpr int kPackShift = 35;               // packed counter: count<<35 | degree sum
constexpr unsigned long long kPackMask = (1ull << kPackShift) - 1;
constexpr int64_t kRowsCap = 1024;           // trace rows per launch
constexpr int kPhaseSlots = 8;               // per-layer barrier timestamps kept for diagnostics
// Frontier bitmaps live in a ring of kPlanes planes, one per depth, so levels
// are stamped once at the end (one coalesced pass) instead of by scattered
// stores at discovery; a plane reused in a deeper traversal is flushed first.
constexpr int kPlanes = 32;
// Column-blocked top-down (hub frontiers): frontier rows are split into
// kCb ranges of target ids and processed range by range so the active slice
// of parent/level/bitmaps/row-starts stays L2-resident.
constexpr int kCbMaxRanges = 32;
constexpr int64_t kCbMaxF = 65536;           // frontier entries eligible for blocking
constexpr int64_t kCbMinArcs = int64_t(1) << 21;
constexpr int64_t kCbMinN = int64_t(1) << 23;
// default range count: one per 2^24 targets, 2..16 (measured: S24 best at 2,
// S28 at 16; S26 — since the expansion does one reduction per arc — at 4-5:
// off 937, 2: 998, 3: 1018, 4: 1025, 5: 1025, 6: 1023, 8: 1018, 16: 1001 GTEPS;
// more ranges add per-range segment overhead)
constexpr int64_t kCbDefaultRanges = 16;
// Top-down layers with at least this many frontier arcs expand fire-and-forget
// and harvest the next frontier from its bitmap (one extra barrier).
constexpr int64_t kHarvestMinArcs = int64_t(1) << 19;
// ... and from this many on the harvest reads the parents instead of a bitmap
// set by a second reduction per arc.
constexpr int64_t kParentHarvestMinArcs = int64_t(1) << 24;

// HB_DCHECK bits (checked builds): 0 parent/level index, 1 bitmap word,
// 2 queue slot, 3 chunk-start slot, 4 adjacency index, 5 column-blocked
// queue, 6 row-start index, 7 level-pass index
struct Ctr {
    unsigned long long packed;  // discovered count << 35 | their degree sum
    unsigned long long gathers;
    unsigned long long fallbacks;
    unsigned long long pad;
};

// Loop state; every CTA keeps an identical replica in registers, CTA 0 also
// persists it here so a traversal can resume across launches.
struct Ctl {
    int64_t layer, v_f, e_f, eu_v, eu_e, prev_vf;
    int32_t dir, kind, done;
    uint32_t lv_done;           // CTAs finished in the level kernel (diagnostics)
    int64_t rows;               // rows written by the last launch
    unsigned long long conv;    // enqueue counter of the bitmap->queue phase
    Ctr ctr[3];
    unsigned long long cbctr[2][kCbMaxRanges];  // per-range segment counters (2 banks)
    unsigned long long work[3];                  // dynamic work counters, slot L%3
};

template <typename OffT>
struct Queue {
    uint32_t *q;   // vertex ids
    OffT *qo;      // exclusive degree prefix
    OffT *qr;      // row starts
    uint32_t *cs;  // chunk starts
    int64_t cap, ncs;  // entries / chunk starts allocated (HB_DCHECK bounds)
};

template <typename OffT>
struct Args {
    const OffT *rs;
    const uint32_t *adj;
    const uint32_t *posw;
    const uint4 *hd;      // head records (common.cuh), rank order over the degree > 0 vertices
    const uint32_t *pre;  // records before bitmap word w (indexed like posw)
    const uint4 *hd2;     // second-tier records (common.cuh), two uint4 per slot
    int64_t n, nw, arcs, ncs;
    int64_t n_pos;        // vertices with degree > 0 (head records)
    uint32_t *parent;
    int32_t *level;
    uint32_t *bits;  // planes vis | B0 | B1 | B2, nw words each
    Queue<OffT> qb[2];
    Queue<OffT> cbq;  // per-range segment queues: entries r*cb_max_f.., chunk starts r*cb_cs_stride..
    int cb_ranges;
    int64_t cb_range_len, cb_cs_stride, cb_min_arcs, harvest_min_arcs, parent_harvest_min_arcs;
    Ctl *ctl;
    hbfs_layer_row *rows;
    unsigned long long *phase_ns;  // kPhaseSlots timestamps per trace row (diagnostics)
    int64_t rows_cap;
    Heur H;
    int max_pos, use_simd, parent_mode, do_init;
    int direct_levels;  // 1: stamp levels at discovery (small graphs), 0: final pass
    int64_t bu_exec_ratio;       // top-down layers run bottom-up when candidates <= ratio * e_f (0: never)
    int64_t part_w0, part_wend;  // partition (PART): owned word range
    int64_t part_lo, part_nown;  // partition (PART): owned vertex range
    uint32_t *cand, *touch;      // partition top-down: remote targets' min parent / touched bits
    int64_t lv_w0, lv_wend;      // bitmap words whose levels this process stamps (all, or a partition's owned words)
    int64_t lv_layers;           // level pass: layer count from the host (partitions), < 0: from the controller state
    int64_t pst[6];              // partition: the global controller state of this layer (layer, v_f, e_f, eu_v, eu_e, prev_vf)
    int32_t pdir;                // partition: the previous layer's direction
    int32_t part_single;         // partition: the only rank (no exchange: queues stay valid across layers)
    unsigned long long *lay_out; // partition: this rank's layer totals {found, degree sum, gathers, fallbacks} (may be null)
    uint32_t root;
};

struct St {
    int64_t layer, v_f, e_f, eu_v, eu_e, prev_vf;
    int dir, kind;
};

struct EnqSmem {
    unsigned long long wtot[kBlock / 32];
    unsigned long long wbase[kBlock / 32];
};

template <typename OffT>
struct TdSmem {
    OffT off[kTdChunk + 2];
    OffT rs[kTdChunk + 2];
    uint32_t u[kTdChunk + 2];
    int64_t q0, cnt, item;
    EnqSmem enq;
};

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Largest index j in [0, len) with a[j] <= x (a non-decreasing, a[0] <= x).
template <typename OffT>
__device__ __forceinline__ int64_t last_le(const OffT *a, int64_t len, uint64_t x) {
    int64_t lo = 0, hi = len;
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if ((uint64_t)a[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

// A bitmap plane (LSB-first words).  Planes are separate arrays: interleaving
// them per word was measured slower (the frontier plane's L1/L2 footprint grows
// 4x and bottom-up probes lose locality).
struct Plane {
    uint32_t *p;
    __device__ __forceinline__ uint32_t &operator[](int64_t w) const { return p[w]; }
};

// Dynamic scheduling: every CTA first takes item blockIdx.x (no atomics, so
// short layers pay nothing), then draws further items from a per-layer counter
// offset past the static range.
__device__ __forceinline__ int64_t block_grab(unsigned long long *work, int64_t *s_item) {
    __syncthreads();
    if (threadIdx.x == 0) *s_item = (int64_t)gridDim.x + (int64_t)atomicAdd(work, 1ull);
    __syncthreads();
    return *s_item;
}

template <typename A_t>
__device__ __forceinline__ Plane depth_plane(const A_t &A, int64_t d) {
    return Plane{A.bits + A.nw * (1 + d % kPlanes)};
}

// Clear the plane that layer L will use as `out` at L+1 (depth L+2), after
// stamping the levels of the depth it held if the ring wrapped (deep graphs).
template <typename A_t>
__device__ __forceinline__ void clear_spare_word(const A_t &A, int64_t L, int64_t w) {
    uint32_t *p = A.bits + A.nw * (1 + (L + 2) % kPlanes) + w;
    if (L + 2 < kPlanes || A.direct_levels) {  // fresh plane / levels already stamped
        *p = 0;
        return;
    }
    uint32_t x = *p;
    if (!x) return;
    if (w >= A.lv_w0 && w < A.lv_wend) {  // (a partition stamps its owned vertices only)
        const int32_t d = (int32_t)(L + 2 - kPlanes);
        while (x) {
            HB_DCHECK(w * 32 + __ffs(x) - 1 < A.n, 0);
            A.level[w * 32 + __ffs(x) - 1] = d;
            x &= x - 1;
        }
    }
    *p = 0;
}

__device__ __forceinline__ bool test_bit(const Plane &bm, uint32_t a) {
    return (bm[a >> 5] >> (a & 31)) & 1u;
}

// Partition mode: is vertex v owned by this rank?
template <bool PART, typename A_t>
__device__ __forceinline__ bool owned_v(const A_t &A, uint32_t v) {
    return !PART || (uint64_t)((int64_t)v - A.part_lo) < (uint64_t)A.part_nown;
}
// Partition mode: a top-down arc into a vertex of another rank: keep the
// smallest parent per target and mark it for the record exchange (csrc/part.cu)
template <typename A_t>
__device__ __forceinline__ void remote_arc(const A_t &A, uint32_t v, uint32_t u) {
    const uint32_t b = 1u << (v & 31);
    atomicMin(&A.cand[v], u);
    if (!(__ldcg(&A.touch[v >> 5]) & b)) atomicOr(&A.touch[v >> 5], b);
}

// Bitmap probe through a raw pointer with a 32-bit word index: one wide
// multiply-add per address instead of a 64-bit add chain.
__device__ __forceinline__ uint32_t ld_global(const uint32_t *gp) {
    uint32_t r;
    asm("ld.global.u32 %0, [%1];" : "=r"(r) : "l"(gp));
    return r;
}
// bm: a global-space address (pin_ptr), so the probe is an explicit LDG.
// HBFS_PROBE_POLICY (profiling builds only): the probe carries an explicit
// L2 evict_normal policy — the default behaviour, made explicit so that ncu's
// per-instruction "L2 Explicit Hit/Miss Policy Evict Normal" counters measure
// the L2 hit rate of the frontier-bitmap probes alone (tools/probe_l2.py).
__device__ __forceinline__ uint32_t probe_word(const uint32_t *__restrict__ bm, uint32_t a) {
#ifdef HBFS_PROBE_POLICY
    uint64_t pol;
    uint32_t r;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    asm("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(bm + (a >> 5)), "l"(pol));
    return r;
#else
    return ld_global(bm + (a >> 5));
#endif
}

// Block-aggregated append to a queue: every thread contributes up to I entries
// (v, deg, row start).  Warps scan their lanes, the CTA scans its warps, and ONE
// 64-bit atomic per CTA reserves both the queue slots and the arc range
// (count<<35 | degree sum), so queue order and arc-prefix order agree and the
// global counter sees one atomic per CTA work item, not one per warp.  Each
// warp also records, for every top-down chunk boundary c*kTdChunk inside its
// arc range, the queue slot holding it — the top-down phase then needs no
// search to start a chunk.  Must be called by every thread of the CTA.
template <typename OffT, int I>
__device__ __forceinline__ void block_enqueue(const bool (&claim)[I], const uint32_t (&v)[I],
                                              const uint64_t (&deg)[I], const OffT (&rsv)[I],
                                              unsigned long long *counter, const Queue<OffT> &Q,
                                              EnqSmem &es) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t cl = 0;
    uint64_t dl = 0;
#pragma unroll
    for (int k = 0; k < I; ++k) {
        cl += claim[k] ? 1u : 0u;
        dl += claim[k] ? deg[k] : 0ull;
    }
    uint32_t ci = cl;
    uint64_t di = dl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t yc = __shfl_up_sync(full, ci, o);
        const uint64_t yd = __shfl_up_sync(full, di, o);
        if (lane >= o) {
            ci += yc;
            di += yd;
        }
    }
    if (lane == 31) es.wtot[wid] = ((unsigned long long)ci << kPackShift) + di;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long run = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            const unsigned long long t = es.wtot[w];
            es.wtot[w] = run;  // exclusive, packed
            run += t;
        }
        es.wbase[0] = run ? atomicAdd(counter, run) : 0ull;
    }
    __syncthreads();
    const unsigned long long wtot = __shfl_sync(full, ((unsigned long long)ci << kPackShift) + di, 31);
    if (wtot == 0) return;
    const unsigned long long base = es.wbase[0] + es.wtot[wid];
    const uint64_t qb = base >> kPackShift, db = base & kPackMask;
    // Queue entries, then the chunk starts inside each entry's arc range
    // (chunk c starts at arc c*kTdChunk): an entry spanning at most two chunk
    // boundaries writes them itself, larger ones (hubs) are written by the
    // whole warp, 32 per step.
    uint64_t pos = qb + ci - cl, off = db + di - dl;
#pragma unroll
    for (int k = 0; k < I; ++k) {
        uint64_t c0 = 0, c1 = 0;
        const uint64_t mypos = pos;
        if (claim[k]) {
            HB_DCHECK(pos < (uint64_t)Q.cap, 2);
            Q.q[pos] = v[k];
            Q.qo[pos] = (OffT)off;
            Q.qr[pos] = rsv[k];
            c0 = (off + kTdChunk - 1) / kTdChunk;
            c1 = (off + deg[k] + kTdChunk - 1) / kTdChunk;
            if (c1 - c0 <= 2)
                for (uint64_t c = c0; c < c1; ++c) {
                    HB_DCHECK(c < (uint64_t)Q.ncs, 3);
                    Q.cs[c] = (uint32_t)pos;
                }
            ++pos;
            off += deg[k];
        }
        unsigned todo = __ballot_sync(full, c1 - c0 > 2);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint64_t b0 = __shfl_sync(full, (unsigned long long)c0, src);
            const uint64_t b1 = __shfl_sync(full, (unsigned long long)c1, src);
            const uint32_t bp = (uint32_t)__shfl_sync(full, (unsigned long long)mypos, src);
            for (uint64_t c = b0 + lane; c < b1; c += 32) {
                HB_DCHECK(c < (uint64_t)Q.ncs, 3);
                Q.cs[c] = bp;
            }
        }
    }
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    return x;
}

// Adjacency vector load with an L2 prefetch-size hint.  Measured on this B200
// (tools/mb/sector.cu under ncu): a plain / .nc / .cs load that misses L2
// fetches the whole 128-byte line from DRAM (dram bytes = 4x the 32-byte
// sector asked for); .L2::64B halves that.  PF = 0: no hint.
template <int PF>
__device__ __forceinline__ uint4 ld_adj4(const uint32_t *p) {
    uint4 r;
    if (PF == 64)
        asm("ld.global.nc.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
            : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if (PF == 128)
        asm("ld.global.nc.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];"
            : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if (PF == 256)
        asm("ld.global.nc.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
            : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else
        r = __ldg(reinterpret_cast<const uint4 *>(p));
    return r;
}

// Row start with the 64-byte L2 fetch hint (a lone 4- or 8-byte read of a line).
template <typename OffT>
__device__ __forceinline__ OffT ld_rs(const OffT *p) {
    if (sizeof(OffT) == 4) {
        uint32_t r;
        asm("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(r) : "l"(p));
        return (OffT)r;
    }
    unsigned long long r;
    asm("ld.global.nc.L2::64B.u64 %0, [%1];" : "=l"(r) : "l"(p));
    return (OffT)r;
}

// Opaque global-space copy of a pointer: the compiler cannot rematerialise it (it would
// otherwise rebuild the bitmap plane address from the parameter bank with a
// 64-bit add chain at every probe — 5 extra instructions per probe).
__device__ __forceinline__ const uint32_t *pin_ptr(const uint32_t *p) {
    const uint32_t *q;
    asm("cvta.to.global.u64 %0, %1;" : "=l"(q) : "l"(p));
    return q;
}

// Frontier probes of a row vector.  The tests are separated from the plane
// loads so that the loads stay independent, predicated instructions.
struct Probe {
    const uint32_t *bm;  // frontier plane (global-space address, pin_ptr)
    __device__ __forceinline__ uint32_t word(uint32_t a) const { return probe_word(bm, a); }
    // N row entries: bit j of the result = val[j] is in the frontier
    template <int N>
    __device__ __forceinline__ uint32_t hitsn(const uint32_t (&val)[N], const bool (&ok)[N]) const {
        uint32_t w[N];
#pragma unroll
        for (int j = 0; j < N; ++j) w[j] = ok[j] ? word(val[j]) : 0u;
        uint32_t hm = 0;
#pragma unroll
        for (int j = 0; j < N; ++j) hm |= ((w[j] >> (val[j] & 31)) & 1u) << j;
        return hm;
    }
    __device__ __forceinline__ uint32_t hits4(const uint32_t (&val)[4], const bool (&ok)[4]) const {
        return hitsn<4>(val, ok);
    }
};

// First hit search of up to 32 rows, one per lane: the first entry of the
// sorted row [s, e) whose bit is set in the frontier plane — the reference's
// first-hit rule (_native.pyx:98-104, bu_probe.h:38-63 + fallback :186-203).
// Each lane first walks its own row for up to `lv` aligned uint4 vectors;
// rows still open are finished cooperatively, lowest position winning (ballot
// + ffs): four rows at a time by 8-lane groups (32 entries per row and step),
// rows with more than kTailLong entries left by the whole warp (128 entries
// per step).  The loops are deliberately not unrolled and the two cooperative
// widths share one body: the bottom-up hot path has to stay inside the 32 KB
// instruction cache (ncu: `no_instruction` stalls dominated a larger variant).
template <typename OffT, int PF = 0>
__device__ __forceinline__ void first_hits(const uint32_t *__restrict__ adj, const Probe &bm,
                                           const bool act, const OffT s, const OffT e, int lv,
                                           int64_t &hit, uint32_t &hu) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    OffT p = s;
    hit = -1;
    hu = 0;
#pragma unroll 1
    for (int it = 0; it < lv; ++it) {
        const bool go = act && hit < 0 && p < e;
        if (!__any_sync(full, go)) break;
        const OffT base = p & ~(OffT)3;
        uint4 q4 = make_uint4(0, 0, 0, 0);
        if (go) q4 = ld_adj4<PF>(adj + base);
        const uint32_t val[4] = {q4.x, q4.y, q4.z, q4.w};
        bool ok[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) ok[j] = go && base + j >= p && base + j < e;
        const uint32_t hm = bm.hits4(val, ok);
        if (go) {
            if (hm) {
                const int j = __ffs(hm) - 1;
                hit = (int64_t)(base + j);
                // select, not val[j]: a dynamic index would put val[] in local memory
                hu = j == 0 ? val[0] : j == 1 ? val[1] : j == 2 ? val[2] : val[3];
            } else {
                p = base + 4;
            }
        }
    }
    const bool open = act && hit < 0 && p < e;
    const unsigned todo_long = __ballot_sync(full, open && (uint64_t)(e - p) > kTailLong);
    const unsigned todo_short = __ballot_sync(full, open) & ~todo_long;
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
        unsigned todo = pass ? todo_long : todo_short;
        const int gsh = pass ? 5 : 3;                  // lanes per row: 8, then 32
        const int gw = 1 << gsh, grp = lane >> gsh, gl = lane & (gw - 1), ng = 32 >> gsh;
        const unsigned gmask = gw == 32 ? ~0u : (1u << gw) - 1u;
        while (todo) {
            unsigned t = todo;
            for (int g = 0; g < grp && t; ++g) t &= t - 1;  // group g takes the g-th open row
            const int src = t ? __ffs(t) - 1 : -1;
            for (int g = 0; g < ng; ++g) todo &= todo - 1;
            const int sl = src < 0 ? 0 : src;
            const OffT ps = __shfl_sync(full, p, sl), pe = __shfl_sync(full, e, sl);
            bool live = src >= 0;
            int64_t h = -1;
            uint32_t hv = 0;
#pragma unroll 1
            for (OffT c = ps & ~(OffT)3;; c += 4 * gw) {
                live = live && c < pe;
                if (!__any_sync(full, live)) break;
                const OffT b4 = c + 4 * gl;
                uint32_t hm = 0;
                uint4 q4 = make_uint4(0, 0, 0, 0);
                if (live && b4 < pe) {
                    q4 = __ldg(reinterpret_cast<const uint4 *>(adj + b4));
                    const uint32_t val[4] = {q4.x, q4.y, q4.z, q4.w};
                    bool ok[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) ok[j] = b4 + j >= ps && b4 + j < pe;
                    hm = bm.hits4(val, ok);
                }
                const unsigned gm = (__ballot_sync(full, hm != 0) >> (grp << gsh)) & gmask;
                const int jm = hm ? __ffs(hm) - 1 : 0;
                const uint32_t mine = jm == 0 ? q4.x : jm == 1 ? q4.y : jm == 2 ? q4.z : q4.w;
                const int wl = gm ? __ffs(gm) - 1 : 0;
                const int srcl = (grp << gsh) + wl;
                const int jw = __shfl_sync(full, jm, srcl);
                const uint32_t vw = __shfl_sync(full, mine, srcl);
                if (live && gm) {
                    h = (int64_t)(c + 4 * wl + jw);
                    hv = vw;
                    live = false;
                }
            }
#pragma unroll 1
            for (int g = 0; g < ng; ++g) {  // results back to the rows' owners
                const int og = __shfl_sync(full, src, g << gsh);
                const int64_t hg = __shfl_sync(full, (long long)h, g << gsh);
                const uint32_t vg = __shfl_sync(full, hv, g << gsh);
                if (lane == og) {
                    hit = hg;
                    hu = vg;
                }
            }
        }
    }
}

// ---------------------------------------------------------------- phases

// a[i] = (i == special ? sv : x) for i in [i0, i1): 16-byte stores over the
// aligned body, scalar head and tail (the buffers may be caller views)
__device__ __forceinline__ void fill_words(uint32_t *a, int64_t i0, int64_t i1, uint32_t x,
                                           int64_t special, uint32_t sv, int64_t tid, int64_t nth) {
    if (i1 <= i0) return;
    int64_t b0 = i0 + (int64_t)((16 - (reinterpret_cast<uintptr_t>(a + i0) & 15)) & 15) / 4;
    if (b0 > i1) b0 = i1;
    const int64_t nv = (i1 - b0) / 4, b1 = b0 + nv * 4;
    for (int64_t i = i0 + tid; i < b0; i += nth) a[i] = i == special ? sv : x;
    for (int64_t i = b1 + tid; i < i1; i += nth) a[i] = i == special ? sv : x;
    uint4 *av = reinterpret_cast<uint4 *>(a + b0);
    for (int64_t q = tid; q < nv; q += nth) {
        uint4 y = make_uint4(x, x, x, x);
        const int64_t r = special - (b0 + 4 * q);
        if ((uint64_t)r < 4) (r == 0 ? y.x : r == 1 ? y.y : r == 2 ? y.z : y.w) = sv;
        av[q] = y;
    }
}

template <typename OffT, bool PART = false>
__device__ void phase_init(const Args<OffT> &A) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const uint32_t root = A.root;
    const int64_t v0 = PART ? A.part_lo : 0, v1 = PART ? A.part_lo + A.part_nown : A.n;
    fill_words(A.parent, v0, v1, HBFS_NIL, (int64_t)root, root, tid, nth);
    if (A.direct_levels)
        fill_words(reinterpret_cast<uint32_t *>(A.level), v0, v1, 0xFFFFFFFFu, (int64_t)root, 0u, tid, nth);
    // vis and B0 hold the root; B1, B2 zero
    const int64_t rw = root >> 5;
    const uint32_t rb = 1u << (root & 31);
    for (int64_t w = tid; w < 3 * A.nw; w += nth)  // vis, depth plane 0 (root), plane 1
        A.bits[w] = (w == rw || w == A.nw + rw) ? rb : 0u;
    if (!PART) {  // partitions convert the root plane instead
        const OffT r0 = __ldg(A.rs + root);
        const uint64_t rdeg = (uint64_t)(__ldg(A.rs + root + 1) - r0);
        const uint64_t nch = (rdeg + kTdChunk - 1) / kTdChunk;
        for (int64_t c = tid; c < (int64_t)nch; c += nth) A.qb[0].cs[c] = 0;
        if (tid == 0) {
            A.qb[0].q[0] = root;
            A.qb[0].qo[0] = 0;
            A.qb[0].qr[0] = r0;
        }
    }
    if (tid == 0) {
        Ctl *c = A.ctl;
        for (int s = 0; s < 3; ++s) {
            c->ctr[s] = Ctr{0, 0, 0, 0};
            c->work[s] = 0;
        }
        for (int b = 0; b < 2; ++b)
            for (int r = 0; r < kCbMaxRanges; ++r) c->cbctr[b][r] = 0;
        c->conv = 0;
        c->done = 0;
        c->lv_done = 0;
    }
}

// Top-down layer: arc-balanced expansion of the frontier queue.  CTA work item =
// kTdChunk consecutive arcs of the concatenated frontier rows, so hubs of any
// degree spread over many CTAs and adjacency reads are coalesced; each thread
// maps its kTdItems arcs to (u, position) by binary search in the CTA's
// shared-memory slice of the degree prefix.  The items are staged (all
// adjacency loads, then all visited-bit loads, then all claims) so their memory
// latencies overlap.  A claim is one atomicOr on the L2-resident visited bitmap;
// the claimer stamps the level and the warp enqueues all its claims with one
// atomic.  Replaces top_down_layer / top_down_chunked (_native.pyx:65-86,
// :207-239).
// Prologue of every top-down layer: clear the spare bitmap; in min-id mode
// commit the frontier to vis (the arc tests use vis | in, so no barrier).
template <typename OffT, bool PART = false>
__device__ void td_prologue(const Args<OffT> &A, const St &S, const Plane spare) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const Queue<OffT> &Q = A.qb[S.layer & 1];
    const Plane vis{A.bits};
    if (PART) {  // also: the all-gathered frontier joins the replicated visited bitmap
        const Plane in = depth_plane(A, S.layer);
        for (int64_t w = tid; w < A.nw; w += nth) {
            clear_spare_word(A, S.layer, w);
            const uint32_t x = in[w];
            if (x && (vis[w] & x) != x) vis[w] |= x;
        }
    } else {
        for (int64_t w = tid; w < A.nw; w += nth) clear_spare_word(A, S.layer, w);
    }
    if (A.parent_mode != HBFS_PARENT_ANY) {
        for (int64_t i = tid; i < S.v_f; i += nth) {
            const uint32_t x = Q.q[i];
            atomicOr(&vis[x >> 5], 1u << (x & 31));
        }
    }
}

// One CTA work item of a top-down layer: kTdChunk consecutive arcs (chunk c of
// nchunks) of the concatenated rows of queue Q (nf entries, mf arcs).  Each
// thread maps its kTdItems arcs to (u, position) by binary search in the CTA's
// shared-memory slice of the degree prefix; the items are staged (all
// adjacency loads, then all visited-bit loads, then all claims) so their
// memory latencies overlap; claims are appended to NQ with one atomic per CTA.
// Harvest=true (large layers): pure fire-and-forget expansion — every arc into
// a vertex unvisited before the layer does RED.OR on its next-frontier bit and
// RED.MIN (min-id) or a plain store (any) on its parent; levels, counters and
// the next queue come from a word-order harvest of the bitmap afterwards.
// SPAN: base chunks (of kTdChunk arcs) per work item; harvest layers use 2.
// Small layers split a chunk into `nsub` sub-items (part `sub`) so that more
// CTAs share it: a single SM's request rate, not latency, bounds a lone chunk.
template <typename OffT, bool Harvest, int SPAN, bool PART = false>
__device__ __forceinline__ void td_chunk(const Args<OffT> &A, const Queue<OffT> &Q, int64_t nf,
                                         uint64_t mf, int64_t c, int64_t nchunks, int32_t depth1,
                                         const Plane in, const Plane out, const Queue<OffT> &NQ,
                                         Ctr *ctr, TdSmem<OffT> &sm, int sub = 0, int nsub = 1,
                                         bool red_out = false) {
    constexpr int I = kTdItems * SPAN;
    const Plane vis{A.bits};
    const bool any_parent = A.parent_mode == HBFS_PARENT_ANY;
        const uint64_t span = (uint64_t)kTdChunk * SPAN / nsub;
        const uint64_t a0 = (uint64_t)c * kTdChunk + (uint64_t)sub * span;
        const uint64_t a1 = min(a0 + span, mf);
        if (threadIdx.x == 0) {
            const int64_t q0 = Q.cs[c];
            const int64_t ql = (c + SPAN < nchunks) ? (int64_t)Q.cs[c + SPAN] : nf - 1;
            sm.q0 = q0;
            sm.cnt = ql - q0 + 1;
        }
        __syncthreads();
        const int64_t q0 = sm.q0, cnt = sm.cnt;
        const bool in_smem = cnt <= kTdChunk + 2;
        if (in_smem) {
            for (int64_t j = threadIdx.x; j < cnt; j += blockDim.x) {
                sm.u[j] = Q.q[q0 + j];
                sm.off[j] = Q.qo[q0 + j];
                sm.rs[j] = Q.qr[q0 + j];
            }
        }
        __syncthreads();
        bool ok[I], claim[I];
        uint32_t v[I], u[I], vw[I];
        uint64_t deg[I];
        OffT rsv[I];
#pragma unroll
        for (int k = 0; k < I; ++k) {
            const uint64_t a = a0 + (uint64_t)k * blockDim.x + threadIdx.x;
            ok[k] = a < a1;
            v[k] = u[k] = 0;
            if (ok[k]) {
                OffT off, rsu;
                if (in_smem) {
                    const int64_t j = last_le(sm.off, cnt, a);
                    off = sm.off[j];
                    u[k] = sm.u[j];
                    rsu = sm.rs[j];
                } else {
                    const int64_t j = q0 + last_le(Q.qo + q0, nf - q0, a);
                    off = Q.qo[j];
                    u[k] = Q.q[j];
                    rsu = Q.qr[j];
                }
                HB_DCHECK((uint64_t)rsu + (a - (uint64_t)off) < (uint64_t)A.arcs, 4);
                v[k] = __ldg(A.adj + (uint64_t)rsu + (a - (uint64_t)off));
                HB_DCHECK(v[k] < A.n && u[k] < A.n, 0);
            }
        }
        if (Harvest) {
            // vis is complete (frontier committed before a barrier) and not
            // written during the expansion: one read-only load per arc, then
            // two reductions without return (next-frontier bit, parent); the
            // harvest pass reads the 1-bit-per-vertex next frontier.
#pragma unroll
            for (int k = 0; k < I; ++k) vw[k] = ok[k] ? __ldg(&vis[v[k] >> 5]) : ~0u;
#pragma unroll
            for (int k = 0; k < I; ++k) {
                const uint32_t b = 1u << (v[k] & 31);
                if (!(vw[k] & b)) {
                    if (!owned_v<PART>(A, v[k])) {
                        remote_arc(A, v[k], u[k]);
                        continue;
                    }
                    // the largest layers: the harvest finds the reached vertices by
                    // their parents (no longer NIL), an arc costs one reduction;
                    // mid-size layers also set the next-frontier bit and harvest
                    // the bitmap (a parent sweep costs more than their reductions)
                    if (red_out) atomicOr(&out[v[k] >> 5], b);
                    if (any_parent) A.parent[v[k]] = u[k];
                    else atomicMin(&A.parent[v[k]], u[k]);
                }
            }
            return;
        } else if (any_parent) {
            // first claimer wins: claim on the visited bitmap itself (one L2
            // load per arc), the claimer also sets the next-frontier bit
#pragma unroll
            for (int k = 0; k < I; ++k) vw[k] = ok[k] ? vis[v[k] >> 5] : ~0u;
#pragma unroll
            for (int k = 0; k < I; ++k) {
                const uint32_t b = 1u << (v[k] & 31);
                claim[k] = false;
                if (!(vw[k] & b)) claim[k] = !(atomicOr(&vis[v[k] >> 5], b) & b);
                if (claim[k]) atomicOr(&out[v[k] >> 5], b);
            }
        } else {
            // min-id parents: every arc into a vertex unvisited before the layer
            // takes part in an atomicMin, so `visited` means "before this layer"
            // (vis | in) and claims go to `out`.
            uint32_t ow[I];
#pragma unroll
            for (int k = 0; k < I; ++k) {
                vw[k] = ok[k] ? (vis[v[k] >> 5] | in[v[k] >> 5]) : ~0u;
                ow[k] = ok[k] ? out[v[k] >> 5] : 0u;
            }
#pragma unroll
            for (int k = 0; k < I; ++k) {
                const uint32_t b = 1u << (v[k] & 31);
                claim[k] = false;
                if (!(vw[k] & b) && !owned_v<PART>(A, v[k])) {
                    remote_arc(A, v[k], u[k]);
                } else if (!(vw[k] & b)) {
                    uint32_t old = ow[k];
                    if (!(old & b)) old = atomicOr(&out[v[k] >> 5], b);
                    claim[k] = !(old & b);
                    atomicMin(&A.parent[v[k]], u[k]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < I; ++k) {
            deg[k] = 0;
            rsv[k] = 0;
            if (claim[k]) {
                if (any_parent) A.parent[v[k]] = u[k];
                if (A.direct_levels) A.level[v[k]] = depth1;
                rsv[k] = __ldg(A.rs + v[k]);
                deg[k] = (uint64_t)(__ldg(A.rs + v[k] + 1) - rsv[k]);
            }
        }
        block_enqueue<OffT, I>(claim, v, deg, rsv, &ctr->packed, NQ, sm.enq);
        __syncthreads();
}

// Top-down layer: arc-balanced expansion of the frontier queue (hubs of any
// degree spread over many CTAs, coalesced adjacency reads).  A claim is one
// atomicOr on an L2-resident bitmap; min-id mode adds atomicMin(parent) for
// every arc into a vertex unvisited before the layer.  Replaces
// top_down_layer / top_down_chunked (_native.pyx:65-86, :207-239).
template <typename OffT, bool Harvest, bool PART = false>
__device__ void phase_td(const Args<OffT> &A, const St &S, const Plane in, const Plane out,
                         const Plane spare, Ctr *ctr, TdSmem<OffT> &sm, bool red_out = false) {
    const Queue<OffT> &Q = A.qb[S.layer & 1];
    const Queue<OffT> &NQ = A.qb[(S.layer + 1) & 1];
    if (!Harvest) td_prologue<OffT, PART>(A, S, spare);  // harvest layers run it before a barrier
    const int64_t nf = S.v_f;
    const uint64_t mf = (uint64_t)S.e_f;
    constexpr int SPAN = Harvest ? 2 : 1;
    const int64_t nchunks = (int64_t)((mf + kTdChunk - 1) / kTdChunk);
    const int64_t nitems = (nchunks + SPAN - 1) / SPAN;
    unsigned long long *work = &A.ctl->work[S.layer % 3];
    int nsub = 1;  // sub-items per chunk on layers with fewer chunks than half the CTAs
    if (!Harvest)
        while (nsub < kTdMaxSub && nitems * nsub * 4 <= (int64_t)gridDim.x) nsub *= 2;
    for (int64_t g = blockIdx.x; g < nitems * nsub; g = block_grab(work, &sm.item))
        td_chunk<OffT, Harvest, SPAN, PART>(A, Q, nf, mf, (g / nsub) * SPAN, nchunks, (int32_t)S.layer + 1,
                                            in, out, NQ, ctr, sm, (int)(g % nsub), nsub, red_out);
}

template <typename OffT>
__device__ __forceinline__ Queue<OffT> cb_queue(const Args<OffT> &A, int r, int64_t cb_max_f) {
    Queue<OffT> q;
    q.q = A.cbq.q + r * cb_max_f;
    q.qo = A.cbq.qo + r * cb_max_f;
    q.qr = A.cbq.qr + r * cb_max_f;
    q.cs = A.cbq.cs + r * A.cb_cs_stride;
    q.cap = cb_max_f;
    q.ncs = A.cb_cs_stride;
    return q;
}

// Column-blocked top-down, phase A: split every frontier row into cb_ranges
// sub-rows by target id (rows are sorted, so each is a contiguous segment
// found by binary search) and append the segments to per-range queues.
template <typename OffT, bool PART = false>
__device__ void phase_cb_build(const Args<OffT> &A, const St &S, const Plane spare, int bank) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const Queue<OffT> &Q = A.qb[S.layer & 1];
    td_prologue<OffT, PART>(A, S, spare);
    const int P = A.cb_ranges;
    const int64_t nf = S.v_f;
    const uint64_t mf = (uint64_t)S.e_f;
    for (int64_t i = tid >> 5; i < nf; i += nth >> 5) {
        const uint32_t u = Q.q[i];
        const OffT s = Q.qr[i];
        const uint64_t o = (uint64_t)Q.qo[i];
        const uint64_t deg = ((i + 1 < nf) ? (uint64_t)Q.qo[i + 1] : mf) - o;
        // lane r: b_r = first row position with target >= r * range_len
        uint64_t b = 0;
        if (lane >= P) b = deg;
        else if (lane > 0) {
            const uint64_t key = (uint64_t)lane * (uint64_t)A.cb_range_len;
            uint64_t lo = 0, hi = deg;
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if ((uint64_t)__ldg(A.adj + (uint64_t)s + mid) < key) lo = mid + 1; else hi = mid;
            }
            b = lo;
        }
        const uint64_t bn = __shfl_down_sync(0xffffffffu, b, 1);
        if (lane < P && bn > b) {
            const uint64_t len = bn - b;
            const unsigned long long old =
                atomicAdd(&A.ctl->cbctr[bank][lane], (1ull << kPackShift) + len);
            const uint64_t pos = old >> kPackShift, db = old & kPackMask;
            const Queue<OffT> R = cb_queue(A, lane, kCbMaxF);
            HB_DCHECK(pos < (uint64_t)kCbMaxF, 5);
            R.q[pos] = u;
            R.qo[pos] = (OffT)db;
            R.qr[pos] = (OffT)((uint64_t)s + b);
            for (uint64_t c = (db + kTdChunk - 1) / kTdChunk; c * kTdChunk < db + len; ++c) {
                HB_DCHECK(c < (uint64_t)A.cb_cs_stride, 5);
                R.cs[c] = (uint32_t)pos;
            }
        }
    }
}

// Column-blocked top-down, phase B: all CTAs walk the chunks of range 0, then
// range 1, ... (one global chunk index space), so the frontier's arcs hit one
// target range at a time.
template <typename OffT, bool Harvest, bool PART = false>
__device__ void phase_cb_run(const Args<OffT> &A, const St &S, const Plane in, const Plane out,
                             Ctr *ctr, int bank, TdSmem<OffT> &sm, int64_t *s_pre, bool red_out = false) {
    const int P = A.cb_ranges;
    const Queue<OffT> &NQ = A.qb[(S.layer + 1) & 1];
    constexpr int SPAN = Harvest ? 2 : 1;
    if (threadIdx.x == 0) {  // prefix of work items (SPAN base chunks each) over ranges
        int64_t run = 0;
        for (int r = 0; r < P; ++r) {
            s_pre[r] = run;
            const unsigned long long t = __ldcg(&A.ctl->cbctr[bank][r]);
            const int64_t nch = (int64_t)(((t & kPackMask) + kTdChunk - 1) / kTdChunk);
            run += (nch + SPAN - 1) / SPAN;
        }
        s_pre[P] = run;
    }
    __syncthreads();
    const int64_t total = s_pre[P];
    int r = 0;
    unsigned long long *work = &A.ctl->work[S.layer % 3];
    for (int64_t g = blockIdx.x; g < total; g = block_grab(work, &sm.item)) {
        while (g >= s_pre[r + 1]) ++r;
        const unsigned long long t = __ldcg(&A.ctl->cbctr[bank][r]);
        const int64_t nf_r = (int64_t)(t >> kPackShift);
        const uint64_t mf_r = t & kPackMask;
        const Queue<OffT> R = cb_queue(A, r, kCbMaxF);
        const int64_t nch_r = (int64_t)((mf_r + kTdChunk - 1) / kTdChunk);
        td_chunk<OffT, Harvest, SPAN, PART>(A, R, nf_r, mf_r, (g - s_pre[r]) * SPAN, nch_r,
                                            (int32_t)S.layer + 1, in, out, NQ, ctr, sm, 0, 1, red_out);
    }
}

// Bottom-up layer.  A warp takes a tile of 32 bitmap words (one per lane), so
// finished words are skipped 32 at a time.  The tile's candidates (unvisited,
// degree > 0) are compacted across the lanes — every lane works regardless of
// how candidates are spread over words — and each lane resolves C candidates
// at once from their 16-byte head records (common.cuh: degree + the first
// kHeadLen row entries): one record load and up to kHeadLen probes of the
// frontier bitmap decide "first hit at position j < kHeadLen" or "row ends
// inside the head, no parent in this layer" without touching the row starts
// or the adjacency array (SCALE 26: 80-99% of the candidates of every
// bottom-up layer, tools/headstats.py).  Candidates still open are pushed on
// a per-warp shared-memory list and drained 32 at a time (one row per lane,
// all lanes busy) by first_hits from row position kHeadLen: uint4 row probes,
// warp-cooperative scan for long rows — the reference's first-hit rule.
// Found bits gather in the warp's shared-memory copy of the tile, then one
// plain store per word updates out/vis (the warp owns its words).  Counters
// gathers/fallbacks are those of the reference's 16-lane kernel.
// Replaces bottom_up_multiple_set / bottom_up_layer (_native.pyx:89-204,
// bu_probe.h:22-106).
// Warp tile scheduler: a warp first walks its own strided share of the leading
// kStaticNum/kStaticDen of the tiles (no atomics: a layer whose tiles are
// mostly empty would otherwise spend its time on one contended counter), then
// draws the remaining tiles one per atomic grab (balances the end of long
// layers).
constexpr int64_t kStaticNum = 7, kStaticDen = 8;
struct TileSched {
    unsigned long long *work;
    int64_t tile, nwarps, nstatic;  // nstatic: tiles handed out statically
    __device__ TileSched(unsigned long long *w, int64_t warp, int64_t nw, int64_t ntiles)
        : work(w), tile(warp), nwarps(nw) {
        const int64_t rounds = ntiles * kStaticNum / kStaticDen / nw;
        nstatic = (rounds > 0 ? rounds : 1) * nw;
    }
    __device__ __forceinline__ int64_t next() {
        if (tile + nwarps < nstatic) return tile += nwarps;
        unsigned long long t = 0;
        if ((threadIdx.x & 31) == 0) t = atomicAdd(work, 1ull);
        tile = nstatic + (int64_t)__shfl_sync(0xffffffffu, t, 0);
        return tile;
    }
};

// Top-down layers over a bitmap frontier run bottom-up when the candidates
// left are at most this many times the frontier's arcs.
constexpr int64_t kBuExecRatio = 2;

constexpr int kOpenCap = 160;  // open-list entries per warp: < 32 pending + one round's pushes (<= 32 * 4)

// Bottom-up shared memory (aliases the top-down staging area, idle then).
// cand: the tile's candidates in vertex order, one 16-bit entry each:
// (rank of the vertex among its word's degree > 0 bits) << 10 | word << 5 | bit.
// open: candidates their head record did not resolve, same entries.
struct BuSmem {
    uint16_t open[kBlock / 32][kOpenCap];
    uint16_t cand[kBlock / 32][1024];
};

// Per-thread packed counters of a bottom-up layer:
// fd = found << 35 | their degree sum; fg = fallbacks << 35 | gathers.
struct BuCount {
    unsigned long long fd = 0, fg = 0;
    __device__ __forceinline__ void add(bool found, int64_t pos, int64_t deg, int64_t max_pos) {
        const bool early = found && pos < max_pos;
        if (found) fd += (1ull << kPackShift) + (unsigned long long)deg;
        fg += (unsigned long long)(early ? pos + 1 : (deg < max_pos ? deg : max_pos));
        if (deg > max_pos && !early) fg += 1ull << kPackShift;
    }
};

// Drain up to 32 open candidates from the top of the warp's list: lane i
// continues row i at position kHeadLen — first in its second-tier record (one
// 32-byte sector: row start + the next 7 entries, 6 with 64-bit offsets), then,
// if the row is longer and still open, in the CSR row itself.
template <typename OffT, int PF>
__device__ __forceinline__ void bu_drain(const Args<OffT> &A, const Probe &bm, const uint16_t *ol,
                                         uint32_t &nopen, int64_t tw, uint32_t prel, uint32_t *s_found,
                                         int64_t max_pos, int32_t depth1, int lv, BuCount &cnt) {
    constexpr int RW = sizeof(OffT) / 4, NE = kH2W - RW;  // second-tier record: row start, then NE entries
    const int lane = threadIdx.x & 31;
    const uint32_t take = nopen < 32u ? nopen : 32u;
    nopen -= take;
    const bool act = (uint32_t)lane < take;
    const uint32_t oe = act ? ol[nopen + lane] : 0u;
    const uint32_t slot = __shfl_sync(0xffffffffu, prel, (oe >> 5) & 31) + (oe >> 10);
    const uint32_t v = (uint32_t)(tw * 32) + (oe & 1023u);
    uint32_t deg = 0;
    uint32_t w[kH2W];
#pragma unroll
    for (int j = 0; j < kH2W; ++j) w[j] = 0;
    if (act) {
        HB_DCHECK(v < A.n, 6);
        deg = __ldg(&A.hd[slot].x);  // a cache hit: the head phase just read the record
        const uint32_t *r2 = reinterpret_cast<const uint32_t *>(A.hd2 + (kH2W / 4) * (int64_t)slot);
#pragma unroll
        for (int q = 0; q < kH2W / 4; ++q) {
            const uint4 r = ld_adj4<PF>(r2 + 4 * q);
            w[4 * q] = r.x;
            w[4 * q + 1] = r.y;
            w[4 * q + 2] = r.z;
            w[4 * q + 3] = r.w;
        }
    }
    const OffT r0 = RW == 2 ? (OffT)(((uint64_t)w[1] << 32) | w[0]) : (OffT)w[0];
    HB_DCHECK(!act || (int64_t)r0 + deg <= A.arcs, 4);
    // the record's entries: row positions kHeadLen .. kHeadLen + NE - 1
    uint32_t val[NE];
    bool ok[NE];
#pragma unroll
    for (int j = 0; j < NE; ++j) {
        val[j] = w[RW + j];
        ok[j] = act && (uint32_t)(kHeadLen + j) < deg;
    }
    const uint32_t hm = bm.template hitsn<NE>(val, ok);
    int64_t hit = -1;
    uint32_t hu = 0;
    if (hm) {
        const int j = __ffs(hm) - 1;
        hit = (int64_t)r0 + kHeadLen + j;
        hu = val[0];  // selects, not val[j]: a dynamic index would put val[] in local memory
#pragma unroll
        for (int i = 1; i < NE; ++i)
            if (j == i) hu = val[i];
    }
    // rows longer than both records that are still open continue in the CSR row
    const bool deep = act && !hm && deg > (uint32_t)(kHeadLen + NE);
    if (__any_sync(0xffffffffu, deep)) {
        const OffT s = (OffT)(r0 + kHeadLen + NE), e = (OffT)(r0 + deg);
        int64_t hit2;
        uint32_t hu2;
        first_hits<OffT, PF>(A.adj, bm, deep, s, e, lv, hit2, hu2);
        if (deep) {
            hit = hit2;
            hu = hu2;
        }
    }
    if (act) {
        const bool found = hit >= 0;
        if (found) {
            HB_DCHECK(hu < A.n && hit < (int64_t)r0 + deg && hit >= (int64_t)r0 + kHeadLen, 0);
            A.parent[v] = hu;
            if (A.direct_levels) A.level[v] = depth1;
            atomicOr(&s_found[(v >> 5) - tw], 1u << (v & 31));
        }
        cnt.add(found, found ? hit - (int64_t)r0 : -1, (int64_t)deg, max_pos);
    }
    __syncwarp();  // the list slots just read may be pushed over
}

// PART: one rank's share of a 1D partition (csrc/part.cu): tiles cover the
// owned words [part_w0, part_wend) only; the arrays indexed by vertex or word
// are offset pointers (see part_bu_launch), and there is no depth ring.
template <typename OffT, int C, bool PART = false, int PF = 0>
__device__ void phase_bu(const Args<OffT> &A, const St &S, const Plane in, const Plane out,
                         const Plane spare, Ctr *ctr, unsigned long long *red, uint32_t *s_found,
                         BuSmem &bs, int lv) {
    uint16_t *ol = bs.open[threadIdx.x >> 5];
    uint16_t *cl = bs.cand[threadIdx.x >> 5];
    const unsigned full = 0xffffffffu;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const Plane vis{A.bits};
    const int64_t max_pos = A.max_pos;
    const int32_t depth1 = (int32_t)S.layer + 1;
    const Probe bm{pin_ptr(in.p)};
    BuCount cnt;
    const int64_t w0 = PART ? A.part_w0 : 0, wend = PART ? A.part_wend : A.nw;
    const int64_t ntiles = (wend - w0 + 31) >> 5;

    TileSched ts(&A.ctl->work[S.layer % 3], tid >> 5, nth >> 5, ntiles);
    for (int64_t tile = ts.tile; tile < ntiles; tile = ts.next()) {
        const int64_t tw = w0 + tile * 32;  // first word of the tile
        const int64_t wl = tw + lane;
        const bool valid = wl < wend;
        const uint32_t vis0 = valid ? vis[wl] : ~0u;
        const uint32_t inl = valid ? in[wl] : 0u;
        const uint32_t pwl = valid ? __ldg(A.posw + wl) : 0u;
        const uint32_t prel = valid ? __ldg(A.pre + wl) : 0u;
        if (!PART && valid) clear_spare_word(A, S.layer, wl);
        const uint32_t vwl = vis0 | inl;
        const uint32_t candl = ~vwl & pwl;
        if (valid && vwl != vis0) vis[wl] = vwl;  // commit a lagging frontier
        const uint32_t cntl = __popc(candl);
        uint32_t incl = cntl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(full, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t T = __shfl_sync(full, incl, 31);
        if (T == 0) continue;
        s_found[lane] = 0;
        // the lane lists its word's candidates at their positions in tile order
        {
            uint32_t pos = incl - cntl;
            for (uint32_t m = candl; m; m &= m - 1) {
                const uint32_t bit = __ffs(m) - 1;
                cl[pos++] = (uint16_t)(__popc(pwl & ((1u << bit) - 1u)) << 10 | lane << 5 | bit);
            }
        }
        __syncwarp();
        // More than one round of candidates: pull the tile's run of head records
        // (contiguous, rank-packed) towards L2 now, so that only the first round
        // waits for DRAM.
        if (T > 32u * C) {
            const uint32_t first = __shfl_sync(full, prel, 0);
            uint32_t npos = __popc(pwl);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) npos += __shfl_xor_sync(full, npos, o);
            const char *slab = reinterpret_cast<const char *>(A.hd + first);
            const uint32_t bytes = npos * (uint32_t)sizeof(uint4);
            for (uint32_t off = lane * 128u; off < bytes; off += 32u * 128u)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(slab + off));
        }
        uint32_t nopen = 0;  // warp-uniform
        for (uint32_t b = 0; b < T; b += 32 * C) {
            bool act[C];
            uint32_t v[C], ce[C];
            uint4 h[C];
#pragma unroll
            for (int k = 0; k < C; ++k) {
                const uint32_t c = b + k * 32 + lane;
                act[k] = c < T;
                const uint32_t ent = ce[k] = act[k] ? cl[c] : 0u;
                v[k] = (uint32_t)(tw * 32) + (ent & 1023u);
                // record slot: rank of v among the degree > 0 vertices
                const uint32_t slot = __shfl_sync(full, prel, (ent >> 5) & 31) + (ent >> 10);
                h[k] = make_uint4(0u, 0u, 0u, 0u);
                if (act[k]) {
                    HB_DCHECK(v[k] < A.n, 6);
                    h[k] = __ldg(A.hd + slot);
                }
            }
            // Probes in two steps: the first head entry alone (it decides most
            // candidates), the other two only where it missed — a probe is a
            // random L2 sector request, and the SM's request rate (about one
            // sector per clock) is what bounds a dense bottom-up layer.
            uint32_t pw[C][kHeadLen];
#pragma unroll
            for (int k = 0; k < C; ++k)  // degree 0 when inactive: no probe
                pw[k][0] = h[k].x > 0 ? bm.word(h[k].y) : 0u;
#pragma unroll
            for (int k = 0; k < C; ++k) {
                const bool more = !((pw[k][0] >> (h[k].y & 31)) & 1u);
                pw[k][1] = more && h[k].x > 1 ? bm.word(h[k].z) : 0u;
                pw[k][2] = more && h[k].x > 2 ? bm.word(h[k].w) : 0u;
            }
#pragma unroll
            for (int k = 0; k < C; ++k) {
                const uint32_t hm = ((pw[k][0] >> (h[k].y & 31)) & 1u) |
                                    (((pw[k][1] >> (h[k].z & 31)) & 1u) << 1) |
                                    (((pw[k][2] >> (h[k].w & 31)) & 1u) << 2);
                const bool found = hm != 0;
                const bool open = act[k] && !found && h[k].x > (uint32_t)kHeadLen;
                if (act[k] && !open) {
                    const int j = __ffs(hm) - 1;  // -1: not found
                    if (found) {
                        const uint32_t hu = j == 0 ? h[k].y : j == 1 ? h[k].z : h[k].w;
                        HB_DCHECK(hu < A.n, 0);
                        A.parent[v[k]] = hu;
                        if (A.direct_levels) A.level[v[k]] = depth1;
                        atomicOr(&s_found[(v[k] >> 5) - tw], 1u << (v[k] & 31));
                    }
                    cnt.add(found, (int64_t)j, (int64_t)h[k].x, max_pos);
                }
                const unsigned m = __ballot_sync(full, open);
                if (open) ol[nopen + __popc(m & lt)] = (uint16_t)ce[k];
                nopen += __popc(m);
            }
            __syncwarp();
            const bool last = b + 32 * C >= T;
            while (nopen >= 32u || (last && nopen))
                bu_drain<OffT, PF>(A, bm, ol, nopen, tw, prel, s_found, max_pos, depth1, lv, cnt);
        }
        __syncwarp();
        const uint32_t f = s_found[lane];
        if (valid && f) {
            out[wl] = f;
            vis[wl] = vwl | f;
        }
        __syncwarp();
    }
    // CTA reduction of the counters, one atomic per CTA per counter.
    unsigned long long c_fd = warp_sum(cnt.fd);
    unsigned long long c_fg = warp_sum(cnt.fg);
    const int wid = threadIdx.x >> 5;
    if (lane == 0) {
        red[wid * 2 + 0] = c_fd;
        red[wid * 2 + 1] = c_fg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t0 = 0, t1 = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            t0 += red[i * 2 + 0];
            t1 += red[i * 2 + 1];
        }
        if (t0) atomicAdd(&ctr->packed, t0);
        if (t1 & kPackMask) atomicAdd(&ctr->gathers, t1 & kPackMask);
        if (t1 >> kPackShift) atomicAdd(&ctr->fallbacks, t1 >> kPackShift);
    }
    __syncthreads();
}

// Block-wide reservation: each thread brings x = count<<35 | degree sum; one
// CTA scan + one atomic on `counter` reserves the queue slots and arc range of
// the whole block; returns the thread's (exclusive) packed base.  Block-uniform.
__device__ __forceinline__ unsigned long long block_reserve(unsigned long long mine,
                                                            unsigned long long *counter,
                                                            EnqSmem &es) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long x = mine;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(full, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) es.wtot[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long run = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            const unsigned long long t = es.wtot[k];
            es.wtot[k] = run;
            run += t;
        }
        es.wbase[0] = run ? atomicAdd(counter, run) : 0ull;
    }
    __syncthreads();
    return es.wbase[0] + es.wtot[wid] + (x - mine);
}

// Append the vertices of bitmap word w (bits) at packed position `base`
// (queue slot << 35 | arc offset): vertex, arc offset, row start, and the
// chunk starts inside its arc range; returns the advanced position.
template <typename OffT>
__device__ __forceinline__ unsigned long long word_append(const Args<OffT> &A, const Queue<OffT> &Q,
                                                          int64_t w, uint32_t bits,
                                                          unsigned long long base) {
    uint64_t pos = base >> kPackShift, off = base & kPackMask;
    while (bits) {
        const uint32_t v = (uint32_t)(w * 32 + __ffs(bits) - 1);
        bits &= bits - 1;
        const OffT r0 = __ldg(A.rs + v);
        const uint64_t d = (uint64_t)(__ldg(A.rs + v + 1) - r0);
        HB_DCHECK(pos < (uint64_t)Q.cap && v < A.n, 2);
        Q.q[pos] = v;
        Q.qo[pos] = (OffT)off;
        Q.qr[pos] = r0;
        for (uint64_t c = (off + kTdChunk - 1) / kTdChunk; c * kTdChunk < off + d; ++c) {
            HB_DCHECK(c < (uint64_t)Q.ncs, 3);
            Q.cs[c] = (uint32_t)pos;
        }
        ++pos;
        off += d;
    }
    return ((unsigned long long)pos << kPackShift) | off;
}

// degree sum of the vertices of word w in `bits`
template <typename OffT>
__device__ __forceinline__ uint64_t word_degsum(const Args<OffT> &A, int64_t w, uint32_t bits) {
    // four vertices per step with their row-start loads issued together
    uint64_t d = 0;
    while (bits) {
        uint32_t v[4];
        bool ok[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            ok[j] = bits != 0;
            v[j] = ok[j] ? (uint32_t)(w * 32 + __ffs(bits) - 1) : 0u;
            bits &= bits - 1;
        }
        OffT a[4], b[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            a[j] = ok[j] ? __ldg(A.rs + v[j]) : (OffT)0;
            b[j] = ok[j] ? __ldg(A.rs + v[j] + 1) : (OffT)0;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) d += (uint64_t)(b[j] - a[j]);
    }
    return d;
}

// Bitmap -> queue (with arc prefix, row starts, chunk starts) at a bottom-up ->
// top-down switch: each thread takes up to kConvWords consecutive words (fewer
// on small graphs, to keep every CTA busy), so a block round covers up to 2048
// words with one reservation; rounds without any frontier bit cost one barrier.
constexpr int kConvWords = 4;

template <typename OffT, bool PART = false>
__device__ void phase_convert(const Args<OffT> &A, const Queue<OffT> &Q, const Plane bm,
                              unsigned long long *counter, bool commit_vis, EnqSmem &es) {
    const Plane vis{A.bits};
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t wa = PART ? A.part_w0 : 0, wb = PART ? A.part_wend : A.nw, nwo = wb - wa;
    const int wpt = nwo >= kConvWords * nth ? kConvWords : (int)(nwo / nth > 1 ? nwo / nth : 1);
    const int64_t span = (int64_t)blockDim.x * wpt;
    for (int64_t b0 = wa + (int64_t)blockIdx.x * span; b0 < wb; b0 += (int64_t)gridDim.x * span) {
        const int64_t w0 = b0 + (int64_t)threadIdx.x * wpt;
        uint32_t bits[kConvWords];
#pragma unroll
        for (int i = 0; i < kConvWords; ++i) bits[i] = i < wpt && w0 + i < wb ? bm[w0 + i] : 0u;
        uint32_t cnt = 0;
        uint64_t dsum = 0;
#pragma unroll
        for (int i = 0; i < kConvWords; ++i) {
            if (!bits[i]) continue;
            if (commit_vis) vis[w0 + i] |= bits[i];
            cnt += __popc(bits[i]);
            dsum += word_degsum(A, w0 + i, bits[i]);
        }
        if (!__syncthreads_or(cnt != 0)) continue;
        unsigned long long base =
            block_reserve(((unsigned long long)cnt << kPackShift) + dsum, counter, es);
        if (!cnt) continue;
#pragma unroll
        for (int i = 0; i < kConvWords; ++i)
            if (bits[i]) base = word_append(A, Q, w0 + i, bits[i], base);
    }
}

// Harvest after a fire-and-forget top-down expansion: a vertex was discovered
// iff it was unvisited before the layer and some frontier arc reached it, i.e.
// iff its parent is no longer NIL.  A warp takes a tile of 32 bitmap words;
// round r reads the parents of word r's unvisited degree > 0 vertices (lane =
// bit: one coalesced 128-byte load) and the ballot of "parent set" is that
// word's share of the next frontier.  Then per word: next-frontier and vis
// words, count and degree sum of the found vertices (and their levels on small
// graphs).  Reading the parents (268 MB at SCALE 26, streamed) instead of a
// next-frontier bitmap set by a second reduction per arc: the expansion is
// bound by the SM's L2 request rate (1 load + 1.5 per reduction, tools/mb).
// Partitions (PART) harvest their owned words the same way.
template <typename OffT, bool PART = false>
__device__ void phase_harvest(const Args<OffT> &A, const Plane out, unsigned long long *counter,
                              unsigned long long *red, int32_t depth1, bool by_bitmap) {
    const Plane vis{A.bits};
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    unsigned long long acc = 0;  // packed count<<35 | degree sum
    const int64_t wa = PART ? A.part_w0 : 0, wb = PART ? A.part_wend : A.nw;
    if (by_bitmap) {
        // mid-size layers: the expansion set the next-frontier bits; thread per
        // word, four words per step with their loads in flight together
        for (int64_t w0 = wa + tid; w0 < wb; w0 += 4 * nth) {
            uint32_t bits[4], vw[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t w = w0 + j * nth;
                bits[j] = w < wb ? __ldcg(&out[w]) : 0u;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) vw[j] = bits[j] ? vis[w0 + j * nth] : 0u;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (!bits[j]) continue;
                const int64_t w = w0 + j * nth;
                vis[w] = vw[j] | bits[j];
                acc += ((unsigned long long)__popc(bits[j]) << kPackShift) + word_degsum(A, w, bits[j]);
                if (A.direct_levels)
                    for (uint32_t x = bits[j]; x; x &= x - 1) {
                        HB_DCHECK(w * 32 + __ffs(x) - 1 < A.n, 0);
                        A.level[w * 32 + __ffs(x) - 1] = depth1;
                    }
            }
        }
    } else {
        const unsigned full = 0xffffffffu;
        const int lane = threadIdx.x & 31;
        const int64_t ntiles = (wb - wa + 31) >> 5;
        for (int64_t tile = tid >> 5; tile < ntiles; tile += nth >> 5) {
            const int64_t tw = wa + tile * 32, wl = tw + lane;
            const bool valid = wl < wb;
            const uint32_t vw = valid ? vis[wl] : ~0u;
            const uint32_t candl = valid ? ~vw & __ldg(A.posw + wl) : 0u;
            uint32_t f = 0;
            if (!__any_sync(full, candl != 0)) continue;
#pragma unroll 1
            for (int r0 = 0; r0 < 32; r0 += 8) {  // 8 words' parent loads in flight together
                // per candidate (lane = bit, so each is one coalesced load per
                // word): its parent and, without waiting for it, its row bounds
                // — the degree counts only if the vertex turns out reached
                uint32_t p[8];
                OffT d[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t cm = __shfl_sync(full, candl, r0 + j);
                    p[j] = HBFS_NIL;
                    d[j] = 0;
                    if ((cm >> lane) & 1u) {
                        const int64_t v = (tw + r0 + j) * 32 + lane;
                        p[j] = __ldcg(A.parent + v);
                        d[j] = __ldg(A.rs + v + 1) - __ldg(A.rs + v);
                    }
                }
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (p[j] == HBFS_NIL) d[j] = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t fm = __ballot_sync(full, p[j] != HBFS_NIL);
                    if (lane == r0 + j) f = fm;
                    acc += (unsigned long long)d[j];
                }
            }
            if (f) {
                out[wl] = f;
                vis[wl] = vw | f;
                acc += (unsigned long long)__popc(f) << kPackShift;
                if (A.direct_levels)
                    for (uint32_t x = f; x; x &= x - 1) {
                        HB_DCHECK(wl * 32 + __ffs(x) - 1 < A.n, 0);
                        A.level[wl * 32 + __ffs(x) - 1] = depth1;
                    }
            }
        }
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
        if (t) atomicAdd(counter, t);
    }
    __syncthreads();
}

// Final level stamp: level[v] = the depth plane holding v (unflushed depths
// d0..nL-1), -1 if never visited; vertices of flushed depths keep the level
// written when their plane was recycled.  A separate kernel launched right
// after the traversal (same stream): it needs the registers the persistent
// kernel cannot spare (all of a word's planes in flight at once) and a plain
// grid with one 32-word tile per warp, so every load of the pass is issued
// up front.  It reads the layer count from the persisted controller state and
// does nothing unless the traversal finished.
constexpr int kLvBlock = 256;
constexpr int kLvBatch = 16;

__device__ __forceinline__ int32_t level_of(uint32_t R, const uint32_t (&D)[5], uint32_t vw,
                                            int64_t d0, int b) {
    uint32_t rel = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) rel |= ((D[k] >> b) & 1u) << k;
    // reached: depth from the planes; visited otherwise: flushed earlier
    return ((R >> b) & 1u) ? (int32_t)(d0 + rel) : (((vw >> b) & 1u) ? -2 : -1);
}

// byte I of x as a sign-extended int32 (prmt with the replicate-sign selector)
template <int I>
__device__ __forceinline__ int32_t sext_byte(uint32_t x) {
    int32_t r;
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(x), "n"(I | (8 | I) << 4 | (8 | I) << 8 | (8 | I) << 12));
    return r;
}

template <typename OffT>
__global__ void __launch_bounds__(kLvBlock) levels_kernel(Args<OffT> A) {
    const Ctl *c = A.ctl;
    if (A.lv_layers < 0 && !__ldcg(&c->done)) return;
    unsigned long long *kstamp = A.phase_ns + kRowsCap * kPhaseSlots;
    if (blockIdx.x == 0 && threadIdx.x == 0) kstamp[3] = globaltimer();
    const int64_t nL = A.lv_layers >= 0 ? A.lv_layers : __ldcg(&c->layer);
    const int64_t lw0 = A.lv_w0, lwend = A.lv_wend;  // words stamped here
    const int lane = threadIdx.x & 31;
    const int64_t d0 = nL + 2 - kPlanes > 0 ? nL + 2 - kPlanes : 0;
    const int64_t ntiles = (lwend - lw0 + 31) / 32;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const bool aligned = (reinterpret_cast<uintptr_t>(A.level) & 15) == 0;
    // lane per word: fold its depth-plane words into binary digit words
    // (bit b of D_k = bit k of the depth of vertex b relative to d0), then the
    // warp writes its tile's 32 words of levels as full 128-byte lines.  Warps
    // walk tiles with a stride and load the next tile's planes before storing
    // the current one (the pass is otherwise a chain of load -> store waves).
    const bool one_batch = nL - d0 <= kLvBatch;
    // next tile's plane rows (and its visited row) stream into shared memory
    // with cp.async while the current tile is folded and stored
    __shared__ uint32_t stage[kLvBlock / 32][2][kLvBatch + 1][32];
    uint32_t(*st)[kLvBatch + 1][32] = stage[threadIdx.x >> 5];
    const int nrow = (int)(nL - d0) + 1;  // planes d0..nL-1, then the visited row
    auto load_tile = [&](int64_t t, int s) {
        const int64_t w = lw0 + t * 32 + lane;
        const unsigned sz = t < ntiles && w < lwend ? 4u : 0u;  // zero-fill past the end
        const int64_t wc = sz ? w : 0;
        for (int j = 0; j < nrow; ++j) {
            const uint32_t *src = j + 1 < nrow ? depth_plane(A, d0 + j).p + wc : A.bits + wc;
            const unsigned dst = (unsigned)__cvta_generic_to_shared(&st[s][j][lane]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(sz) : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    int s = 0;
    if (one_batch) load_tile(warp, 0);
    for (int64_t t = warp; t < ntiles; t += nwarps, s ^= 1) {
        const int64_t w = lw0 + t * 32 + lane;
        uint32_t R = 0, D[5] = {0, 0, 0, 0, 0}, vw;
        if (one_batch) {
            load_tile(t + nwarps, s ^ 1);  // in flight while this tile is stored
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
            __syncwarp();
            for (int j = 0; j + 1 < nrow; ++j) {
                const uint32_t p = st[s][j][lane];
                R |= p;
#pragma unroll
                for (int k = 0; k < 5; ++k) D[k] |= ((j >> k) & 1) ? p : 0u;
            }
            vw = st[s][nrow - 1][lane];
            __syncwarp();  // stage s is refilled next iteration
        } else {  // deep traversals: all held planes, batch by batch
            vw = w < lwend ? __ldcs(A.bits + w) : 0u;
            for (int64_t g0 = d0; g0 < nL; g0 += kLvBatch) {
                uint32_t p[kLvBatch];
#pragma unroll
                for (int j = 0; j < kLvBatch; ++j)
                    p[j] = w < lwend && g0 + j < nL ? __ldcs(depth_plane(A, g0 + j).p + w) : 0u;
#pragma unroll
                for (int j = 0; j < kLvBatch; ++j) {
                    const uint32_t rel = (uint32_t)(g0 + j - d0);
                    R |= p[j];
#pragma unroll
                    for (int k = 0; k < 5; ++k) D[k] |= ((rel >> k) & 1u) ? p[j] : 0u;
                }
            }
        }
        const bool fast = d0 == 0 && lw0 + t * 32 + 32 <= lwend && (lw0 + t * 32 + 32) * 32 <= A.n &&
                          aligned;  // warp-uniform
        if (fast) {
            // round r: the warp writes words 4r..4r+3 of the tile (512
            // contiguous bytes, four full lines); lane l takes levels
            // 4(l%8)..+3 of word 4r + l/8.  Nothing is flushed (d0 = 0), so
            // visited implies reached and a level is its 5 digit bits: the
            // four vertices' digit nibbles are spread one bit per byte
            // (x * 0x00204081 puts bit i at byte i), unreached bytes become
            // 0xFF, and a sign-extending byte permute widens each to int32.
            const int b0 = 4 * (lane & 7);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int src = 4 * r + (lane >> 3);
                uint32_t v = 0;
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    const uint32_t nib = (__shfl_sync(0xffffffffu, D[k], src) >> b0) & 0xFu;
                    v |= (nib * (0x00204081u << k)) & (0x01010101u << k);
                }
                const uint32_t hit = (((__shfl_sync(0xffffffffu, R, src) >> b0) & 0xFu) * 0x00204081u) & 0x01010101u;
                v |= (hit ^ 0x01010101u) * 0xFFu;
                HB_DCHECK((lw0 + t * 32 + src) * 32 + 32 <= A.n, 7);
                int4 *gdst = reinterpret_cast<int4 *>(A.level + (lw0 + t * 32 + src) * 32);
                __stcs(gdst + (lane & 7), make_int4(sext_byte<0>(v), sext_byte<1>(v), sext_byte<2>(v), sext_byte<3>(v)));
            }
        } else if (w < lwend) {
            int32_t *dst = A.level + w * 32;
            HB_DCHECK(w < A.nw, 7);
            for (int b = 0; b < 32; ++b) {
                const int32_t lv = level_of(R, D, vw, d0, b);
                if (w * 32 + b < A.n && lv != -2) dst[b] = lv;
            }
        }
    }
    // last CTA out stamps the end of the pass (diagnostics)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&A.ctl->lv_done, 1u) == gridDim.x - 1) {
            kstamp[4] = globaltimer();
            A.ctl->lv_done = 0;
        }
    }
}

// K: first-hit searches in flight per lane in the bottom-up phase;
// MINB: CTAs per SM the register allocation must allow.
// SCAN: also compile the 4-vector bottom-up path for tiny-frontier layers
// (large graphs only; it costs registers on the small-graph variant).
// PART: one layer of one rank's share of a 1D partition per launch (the host
// loop in csrc/part.cu exchanges records and frontier slices between launches
// and writes the global controller state into ctl); min-id parents, levels
// stamped at discovery, the frontier queue always rebuilt from the owned words.
template <typename OffT, int K, int MINB, bool SCAN, bool PART = false>
__global__ void __launch_bounds__(kBlock, MINB) bfs_kernel(Args<OffT> A) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char dsm[];
    TdSmem<OffT> &sm = *reinterpret_cast<TdSmem<OffT> *>(dsm);
    __shared__ unsigned long long red[(kBlock / 32) * 4];
    __shared__ uint32_t s_found[kBlock];  // per warp: found bits of its 32-word tile
    __shared__ int64_t s_pre[kCbMaxRanges + 1];
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;

    St S;
    unsigned long long *kstamp = A.phase_ns + kRowsCap * kPhaseSlots;  // kernel-level marks
    if (leader) kstamp[0] = globaltimer();
    if (A.do_init) {
        phase_init<OffT, PART>(A);
        grid.sync();
        if (leader) kstamp[1] = globaltimer();
    }
    if (A.do_init && !PART) {
        const int64_t rdeg = (int64_t)(__ldg(A.rs + A.root + 1) - __ldg(A.rs + A.root));
        S.layer = 0;
        S.v_f = 1;
        S.e_f = rdeg;
        S.eu_v = A.n - 1;
        S.eu_e = A.arcs - rdeg;
        S.prev_vf = 0;
        S.dir = HBFS_TOP_DOWN;
        S.kind = 0;
    } else if (PART) {  // the global state, from the host loop
        S.layer = A.pst[0];
        S.v_f = A.pst[1];
        S.e_f = A.pst[2];
        S.eu_v = A.pst[3];
        S.eu_e = A.pst[4];
        S.prev_vf = A.pst[5];
        S.dir = A.pdir;
        // the frontier arrives as an all-gathered bitmap; a single-rank partition
        // keeps the queue its own claim path built (as on one GPU)
        S.kind = A.part_single && !A.do_init ? __ldcg(&A.ctl->kind) : 1;
    } else {  // resumed
        const Ctl *c = A.ctl;
        S.layer = __ldcg(&c->layer);
        S.v_f = __ldcg(&c->v_f);
        S.e_f = __ldcg(&c->e_f);
        S.eu_v = __ldcg(&c->eu_v);
        S.eu_e = __ldcg(&c->eu_e);
        S.prev_vf = __ldcg(&c->prev_vf);
        S.dir = __ldcg(&c->dir);
        S.kind = __ldcg(&c->kind);
    }

    int64_t rows = 0;
    uint64_t t_start = leader ? globaltimer() : 0;
#define STAMP(k) \
    if (leader) A.phase_ns[rows * kPhaseSlots + (k)] = globaltimer()
    while (S.v_f > 0 && rows < A.rows_cap) {
        if (leader)
            for (int k = 0; k < kPhaseSlots; ++k) A.phase_ns[rows * kPhaseSlots + k] = 0;
        STAMP(0);
        int64_t fv, gv;
        const int dir = decide(A.H, S.dir, S.v_f, S.e_f, S.eu_v, S.eu_e, S.prev_vf, &fv, &gv);
        const int64_t L = S.layer;
        const Plane in = depth_plane(A, L), out = depth_plane(A, L + 1),
                    spare = depth_plane(A, L + 2);
        Ctr *ctr = &A.ctl->ctr[L % 3];
        // SQ: the frontier queue's size (the layer's counts on one GPU; the
        // rank's own share, from the conversion, in a partition)
        St SQ = S;
        // How the layer is executed (the trace reports `dir`): a top-down layer
        // whose frontier is only a bitmap (it follows a bottom-up or harvest
        // layer) would first convert it to a queue, an O(n) sweep like a
        // bottom-up layer's; when few candidates are left — unvisited vertices
        // with degree > 0 — the bottom-up sweep alone is cheaper and finds the
        // same vertices with the same parents (first hit in a sorted row =
        // smallest frontier neighbour).  SCALE 26: such layers 100-200 -> 30 us.
        int xdir = dir;
        // (partitions: the frontier is always a bitmap, the sweep stays local to
        // the rank, and the host loop takes the same decision — bu_executes — to
        // skip the record exchange)
        if (bu_executes(xdir, S.kind, S.eu_v, S.e_f, A.n, A.n_pos, A.bu_exec_ratio)) xdir = HBFS_BOTTOM_UP;
        if (xdir == HBFS_TOP_DOWN && S.kind == 1) {
            phase_convert<OffT, PART>(A, A.qb[L & 1], in, &A.ctl->conv, false, sm.enq);
            grid.sync();
            STAMP(1);
            if (PART) {
                const unsigned long long cv = __ldcg(&A.ctl->conv);
                SQ.v_f = (int64_t)(cv >> kPackShift);
                SQ.e_f = (int64_t)(cv & kPackMask);
            }
        }
        const bool cb = xdir == HBFS_TOP_DOWN && A.cb_ranges > 1 && SQ.e_f >= A.cb_min_arcs &&
                        SQ.v_f <= kCbMaxF;
        // Slot (L+1)%3 was last read right after the barrier that ended layer
        // L-2, so every CTA is past that read; it must be zero when layer L+1
        // starts accumulating.  The conversion counter is free again too.
        if (leader) {
            A.ctl->ctr[(L + 1) % 3] = Ctr{0, 0, 0, 0};
            A.ctl->work[(L + 1) % 3] = 0;
            if (!PART) A.ctl->conv = 0;  // PART: reset at the end of the layer (other CTAs read it above)
            for (int r = 0; r < kCbMaxRanges; ++r) A.ctl->cbctr[(L + 1) & 1][r] = 0;
        }
        // Top-down regimes by frontier arcs: claim path (builds the next queue),
        // from harvest_min_arcs fire-and-forget expansion + harvest — of the
        // next-frontier bitmap set by a second reduction per arc, or, from
        // parent_harvest_min_arcs, of the parents (one reduction per arc, but a
        // sweep over every unvisited vertex's parent).
        const bool harvest = xdir == HBFS_TOP_DOWN && SQ.e_f >= A.harvest_min_arcs;
        const bool red_out = harvest && SQ.e_f < A.parent_harvest_min_arcs;
        if (cb) {
            phase_cb_build<OffT, PART>(A, SQ, spare, (int)(L & 1));
            grid.sync();
            STAMP(2);
            if (harvest) phase_cb_run<OffT, true, PART>(A, SQ, in, out, ctr, (int)(L & 1), sm, s_pre, red_out);
            else phase_cb_run<OffT, false, PART>(A, SQ, in, out, ctr, (int)(L & 1), sm, s_pre);
        } else if (xdir == HBFS_TOP_DOWN) {
            if (harvest) {
                td_prologue<OffT, PART>(A, SQ, spare);
                grid.sync();  // vis now holds the frontier: the expansion tests vis alone
                STAMP(2);
                phase_td<OffT, true, PART>(A, SQ, in, out, spare, ctr, sm, red_out);
            } else {
                phase_td<OffT, false, PART>(A, SQ, in, out, spare, ctr, sm);
            }
        }
        if (harvest) {
            grid.sync();
            STAMP(3);
            phase_harvest<OffT, PART>(A, out, &ctr->packed, red, (int32_t)L + 1, red_out);
        }
        if (xdir == HBFS_BOTTOM_UP) {
            uint32_t *sf = s_found + (threadIdx.x & ~31);
            const Plane vis_all{A.bits};
            if (PART) {  // the owned-word tiles do not cover the replicated planes:
                // clear the spare plane; absorb the all-gathered frontier into
                // the other ranks' words of vis (owned words: phase_bu's commit)
                const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
                for (int64_t w = tid; w < A.nw; w += (int64_t)gridDim.x * blockDim.x) {
                    clear_spare_word(A, S.layer, w);
                    if (w >= A.part_w0 && w < A.part_wend) continue;
                    const uint32_t x = in[w];
                    if (x && (vis_all[w] & x) != x) vis_all[w] |= x;
                }
            }
            BuSmem &bs = *reinterpret_cast<BuSmem *>(dsm);  // the top-down staging area is idle
            // rows walked per lane before the cooperative scan: 2 vectors, 4 behind
            // a small frontier (there most open rows are scanned to their end)
            // (large graphs: an open row's vector that misses L2 fetches 64 bytes, not
            // the 128-byte line — tools/mb/sector.cu — most rows stop within it)
            phase_bu<OffT, K, PART, SCAN ? 64 : 0>(A, S, in, out, spare, ctr, red, sf, bs,
                                    SCAN && S.v_f * 64 < A.n ? kLaneVecsScan : kLaneVecs);
        }
        grid.sync();

        STAMP(4);
        const unsigned long long packed = __ldcg(&ctr->packed);
        const int64_t nvf = (int64_t)(packed >> kPackShift);
        const int64_t nef = (int64_t)(packed & kPackMask);
        if (leader) {
            const uint64_t now = globaltimer();
            hbfs_layer_row r;
            r.layer = (int32_t)(L + 1);
            r.direction = dir;
            r.v_f = S.v_f;
            r.e_f = S.e_f;
            r.e_u = A.H.counter_mode ? S.eu_e : S.eu_v;
            r.f_value = fv;
            r.g_value = gv;
            if (!A.use_simd) {
                r.fallback_count = 0;
                r.gather_count = 0;
            } else if (dir == HBFS_TOP_DOWN) {
                r.fallback_count = 0;
                r.gather_count = S.e_f;  // 16-lane chunks incl. tail = frontier degree sum
            } else {
                r.fallback_count = (int64_t)__ldcg(&ctr->fallbacks);
                r.gather_count = (int64_t)__ldcg(&ctr->gathers);
            }
            r.elapsed = (double)(now - t_start) * 1e-9;
            A.rows[rows] = r;
            t_start = now;
            if (PART) {
                A.ctl->conv = 0;  // every CTA read it barriers ago; free for the next launch
                if (A.lay_out) {  // this rank's totals, for the host loop's single read-back
                    A.lay_out[0] = (unsigned long long)nvf;
                    A.lay_out[1] = (unsigned long long)nef;
                    A.lay_out[2] = __ldcg(&ctr->gathers);
                    A.lay_out[3] = __ldcg(&ctr->fallbacks);
                }
            }
        }
        S.prev_vf = S.v_f;
        S.v_f = nvf;
        S.e_f = nef;
        S.eu_v -= nvf;
        S.eu_e -= nef;
        S.dir = dir;
        S.kind = (xdir == HBFS_TOP_DOWN && !harvest) ? 0 : 1;  // harvest and bottom-up build no queue
        S.layer = L + 1;
        ++rows;
    }
    if (leader) kstamp[2] = globaltimer();
    if (leader) {
        Ctl *c = A.ctl;
        c->layer = S.layer;
        c->v_f = S.v_f;
        c->e_f = S.e_f;
        c->eu_v = S.eu_v;
        c->eu_e = S.eu_e;
        c->prev_vf = S.prev_vf;
        c->dir = S.dir;
        c->kind = S.kind;
        c->rows = rows;
        c->done = S.v_f == 0;
    }
}

// ------------------------------------------------- partition bottom-up

// One rank's bottom-up layer with the persistent kernel's tile machinery
// (phase_bu<PART>): called by hbfs_part_bu (csrc/part.cu) as a plain launch.
template <typename OffT, int K>
__global__ void __launch_bounds__(kBlock, 2) part_bu_kernel(Args<OffT> A, St S, Ctr *ctr, const uint32_t *inp,
                                                          uint32_t *outp, int lv) {
    __shared__ unsigned long long red[(kBlock / 32) * 4];
    __shared__ uint32_t s_found[kBlock];
    __shared__ BuSmem bs;
    phase_bu<OffT, K, true>(A, S, Plane{const_cast<uint32_t *>(inp)}, Plane{outp}, Plane{nullptr},
                            ctr, red, s_found + (threadIdx.x & ~31), bs, lv);
}

// Ctr (found << 35 | degree sum, gathers, fallbacks) -> {found, degree sum, gathers, fallbacks}
__global__ void part_bu_counters(const Ctr *c, unsigned long long *out) {
    out[0] = c->packed >> kPackShift;
    out[1] = c->packed & kPackMask;
    out[2] = c->gathers;
    out[3] = c->fallbacks;
}

size_t part_bu_scratch_bytes() { return sizeof(Ctl) + 64; }

int part_bu_launch(const uint64_t *rs_local, const uint32_t *adj, const uint32_t *posw_local,
                   const uint4 *hd_local, int64_t n_pos_local, const uint32_t *pre_local, int64_t n,
                   int64_t lo, int64_t nloc, int64_t arcs_local, const uint32_t *F, uint32_t *V, uint32_t *parent_local,
                   int32_t *level_local, uint32_t *next_slice, int32_t depth, int32_t max_pos, int64_t v_f,
                   unsigned long long *counters, void *scratch, cudaStream_t st) {
    const int64_t wlo = lo >> 5, wown = (nloc + 31) / 32;
    Args<uint64_t> A;
    memset(&A, 0, sizeof(A));
    // vertex- and word-indexed arrays are offset so that global ids index them
    A.rs = rs_local - lo;
    A.adj = adj;
    A.posw = posw_local - wlo;
    A.hd = hd_local;  // rank order within the partition
    A.hd2 = hd_local + head2_offset(n_pos_local);
    A.pre = pre_local - (lo >> 5);
    A.n = n;
    A.nw = (n + 31) / 32;
    A.arcs = arcs_local;
    A.parent = parent_local - lo;
    A.level = level_local - lo;
    A.bits = V;
    A.direct_levels = 1;
    A.max_pos = max_pos;
    A.ctl = static_cast<Ctl *>(scratch);
    A.part_w0 = wlo;
    A.part_wend = wlo + wown;
    St S;
    memset(&S, 0, sizeof(S));
    S.layer = depth;
    S.v_f = v_f;
    Ctr *ctr = &A.ctl->ctr[0];
    HB_CUDA(cudaMemsetAsync(scratch, 0, sizeof(Ctl), st));
    static int grid = 0;
    if (!grid) {
        int per_sm = 0, sms = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        HB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, part_bu_kernel<uint64_t, 2>,
                                                              kBlock, 0));
        grid = std::max(1, per_sm) * sms;
    }
    uint32_t *outp = next_slice - wlo;
    // tiny frontier: rows are mostly scanned to their end
    part_bu_kernel<uint64_t, 2><<<grid, kBlock, 0, st>>>(A, S, ctr, F, outp,
                                                        v_f >= 0 && v_f * 64 < n ? kLaneVecsScan : kLaneVecs);
    part_bu_counters<<<1, 1, 0, st>>>(ctr, counters);
    HB_CUDA(cudaGetLastError());
    return HBFS_OK;
}

// ------------------------------------------------------------ variants

// Kernel variants compiled into the library (occupancy/MLP trade-offs);
// HBFS_KERNEL_VARIANT=<index> selects one, default kDefaultVariant.
template <typename OffT>
struct Variant {
    const void *fn;
    int k, minb;
};

template <typename OffT>
static const Variant<OffT> *variants(int *count) {
    static const Variant<OffT> v[] = {
        {(const void *)bfs_kernel<OffT, 2, 1, false>, 2, 1},
        {(const void *)bfs_kernel<OffT, 1, 1, false>, 1, 1},
        {(const void *)bfs_kernel<OffT, 1, 2, true>, 1, 2},
        {(const void *)bfs_kernel<OffT, 2, 2, true>, 2, 2},
        {(const void *)bfs_kernel<OffT, 4, 1, false>, 4, 1},
        {(const void *)bfs_kernel<OffT, 3, 2, true>, 3, 2},
        {(const void *)bfs_kernel<OffT, 4, 2, true>, 4, 2},
    };
    *count = (int)(sizeof(v) / sizeof(v[0]));
    return v;
}
constexpr int kDefaultVariant = 0;

// Measured on B200 (tools/diag.py sweeps): small graphs are latency-bound and
// prefer one fat CTA per SM with 4 head records in flight per lane (variant 4);
// from 2^22 vertices on two CTAs per SM with 3 per lane win (variant 5; S26, 32
// roots: 2 per lane 1041, 3: 1060, 4: 1046 GTEPS; variant 4 / 5 at S21 311 / 258,
// S22 407 / 412, S23 526 / 564, uniform 2^21 213 / 186, uniform 2^22 231 / 253).

static int variant_index(int64_t n) {
    const char *e = getenv("HBFS_KERNEL_VARIANT");
    if (e) return atoi(e);
    return n >= (int64_t(1) << 22) ? 5 : 4;
}

// ------------------------------------------------------------ workspace

struct Workspace {
    int64_t n = 0;
    int wide = 0;
    DevBuf parent, level, bits, q, qo, qr, cs, ctl;  // ctl: Ctl followed by kRowsCap rows
    DevBuf phases;  // kRowsCap * kPhaseSlots barrier timestamps (last launch)
    DevBuf cbq, cbqo, cbqr, cbcs;  // column-blocked top-down segment queues
    int cb_ranges = 0;
    int64_t ncs = 0;  // chunk-start entries per queue buffer
    int grid = 0, lv_grid = 0;
    size_t smem = 0;
    const void *fn = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    void *h_ctl = nullptr;  // pinned mirror of ctl + rows
    ~Workspace() {
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (h_ctl) cudaFreeHost(h_ctl);
    }
};

static int64_t env_i64(const char *name, int64_t dflt) {
    const char *e = getenv(name);
    return e ? atoll(e) : dflt;
}

int64_t bu_exec_ratio() { return env_i64("HBFS_BU_EXEC_RATIO", kBuExecRatio); }

template <typename OffT>
static size_t dyn_smem_bytes() {
    size_t b = sizeof(TdSmem<OffT>);  // top-down phases; bottom-up: open lists + candidate lists
    if (sizeof(BuSmem) > b) b = sizeof(BuSmem);
    return (b + 15) & ~(size_t)15;
}


static size_t ctl_bytes() { return sizeof(Ctl) + kRowsCap * sizeof(hbfs_layer_row); }

template <typename OffT>
static int ws_alloc(hbfs_graph *g) {
    if (g->ws) return HBFS_OK;
    Workspace *w = new Workspace();
    const int64_t n = g->n, nw = g->nw;
    int rc = HBFS_OK;
    if (!rc) rc = w->parent.alloc(n * 4);
    if (!rc) rc = w->level.alloc(n * 4);
    w->ncs = g->arcs / kTdChunk + 2;
    if (!rc) rc = w->bits.alloc((1 + kPlanes) * nw * 4 + 64);
    if (!rc) rc = w->q.alloc(2 * (n + 1) * 4 + 16);
    if (!rc) rc = w->qo.alloc(2 * (n + 1) * sizeof(OffT));
    if (!rc) rc = w->qr.alloc(2 * (n + 1) * sizeof(OffT));
    if (!rc) rc = w->cs.alloc(2 * w->ncs * 4);
    // column blocking for graphs whose parent/level arrays exceed L2
    // (HBFS_CB_MIN_N / HBFS_CB_RANGES: test knobs that force blocking on small graphs)
    const int64_t cb_min_n = env_i64("HBFS_CB_MIN_N", kCbMinN);
    w->cb_ranges = n >= cb_min_n ? (int)std::min<int64_t>(kCbDefaultRanges, std::max<int64_t>(2, n >> 24)) : 0;
    if (w->cb_ranges) w->cb_ranges = (int)std::min<int64_t>(31, env_i64("HBFS_CB_RANGES", w->cb_ranges));
    if (!rc && w->cb_ranges) {
        const int64_t P = w->cb_ranges;
        rc = w->cbq.alloc(P * kCbMaxF * 4);
        if (!rc) rc = w->cbqo.alloc(P * kCbMaxF * sizeof(OffT));
        if (!rc) rc = w->cbqr.alloc(P * kCbMaxF * sizeof(OffT));
        if (!rc) rc = w->cbcs.alloc(P * w->ncs * 4);
    }
    if (!rc) rc = w->ctl.alloc(ctl_bytes());
    if (!rc) rc = w->phases.alloc((kRowsCap + 1) * kPhaseSlots * 8);
    if (!rc && cudaMallocHost(&w->h_ctl, ctl_bytes()) != cudaSuccess)
        rc = set_error(HBFS_ECUDA, "cudaMallocHost failed");
    if (!rc && (cudaEventCreate(&w->ev0) != cudaSuccess || cudaEventCreate(&w->ev1) != cudaSuccess))
        rc = set_error(HBFS_ECUDA, "cudaEventCreate failed");
    if (!rc) {
        int per_sm = 0, sms = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        int nv = 0;
        const Variant<OffT> *vt = variants<OffT>(&nv);
        int vi = variant_index(n);
        if (vi < 0 || vi >= nv) vi = kDefaultVariant;
        w->fn = vt[vi].fn;
        w->smem = dyn_smem_bytes<OffT>() + (size_t)env_i64("HBFS_SMEM_PAD", 0);  // experiment knob
        cudaError_t e = cudaFuncSetAttribute(w->fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)w->smem);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, w->fn, kBlock, w->smem);
        if (e != cudaSuccess || per_sm < 1)
            rc = set_error(HBFS_ECUDA, "occupancy query failed: %s", cudaGetErrorString(e));
        w->grid = (int)(std::min<int64_t>(per_sm, env_i64("HBFS_GRID_PER_SM", per_sm)) *
                        std::min<int64_t>(sms, env_i64("HBFS_GRID_SMS", sms)));
        int lv_per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&lv_per_sm, levels_kernel<OffT>, kLvBlock, 0);
        w->lv_grid = std::max(1, lv_per_sm) * sms * (int)env_i64("HBFS_LV_WAVES", 1);
    }
    if (rc) {
        delete w;
        return rc;
    }
    w->n = n;
    w->wide = g->wide;
    g->ws = w;
    return HBFS_OK;
}

template <typename OffT>
static int run_bfs(hbfs_graph *g, uint32_t root, const hbfs_params *p, uint32_t *parent,
                   int32_t *level, int on_device, hbfs_layer_row *trace, int64_t trace_cap,
                   int64_t *n_layers, float *device_ms, cudaStream_t st) {
    HB_CHECK(ws_alloc<OffT>(g));
    Workspace *w = g->ws;
    Args<OffT> A;
    A.rs = g->rs.as<OffT>();
    A.adj = g->adj.as<uint32_t>();
    A.posw = g->posw.as<uint32_t>();
    A.hd = g->hd.as<uint4>();
    A.hd2 = g->hd.as<uint4>() + head2_offset(g->n_pos);
    A.lv_w0 = 0;
    A.lv_wend = g->nw;
    A.lv_layers = -1;
    A.pre = g->pre.as<uint32_t>();
    A.n_pos = g->n_pos;
    A.bu_exec_ratio = bu_exec_ratio();
    A.n = g->n;
    A.nw = g->nw;
    A.arcs = g->arcs;
    const bool dev_out = on_device != 0;
    A.parent = (dev_out && parent) ? parent : w->parent.as<uint32_t>();
    A.level = (dev_out && level) ? level : w->level.as<int32_t>();
    A.bits = w->bits.as<uint32_t>();
    A.ncs = w->ncs;
    A.cb_ranges = w->cb_ranges;
    A.cb_range_len = w->cb_ranges ? (g->n + w->cb_ranges - 1) / w->cb_ranges : 0;
    A.cb_cs_stride = w->ncs;
    A.cb_min_arcs = env_i64("HBFS_CB_MIN_ARCS", kCbMinArcs);
    A.harvest_min_arcs = env_i64("HBFS_HARVEST_MIN_ARCS", kHarvestMinArcs);
    A.parent_harvest_min_arcs = env_i64("HBFS_PARENT_HARVEST_MIN_ARCS", kParentHarvestMinArcs);
    // level arrays that fit L2 take scattered stores cheaply; larger graphs
    // stamp levels once from the depth planes (HBFS_DEFER_LEVELS_MIN_N: test knob)
    A.direct_levels = g->n < env_i64("HBFS_DEFER_LEVELS_MIN_N", int64_t(1) << 22);
    A.cbq.q = w->cbq.as<uint32_t>();
    A.cbq.qo = w->cbqo.as<OffT>();
    A.cbq.qr = w->cbqr.as<OffT>();
    A.cbq.cs = w->cbcs.as<uint32_t>();
    for (int b = 0; b < 2; ++b) {
        A.qb[b].q = w->q.as<uint32_t>() + b * (g->n + 1);
        A.qb[b].qo = w->qo.as<OffT>() + b * (g->n + 1);
        A.qb[b].qr = w->qr.as<OffT>() + b * (g->n + 1);
        A.qb[b].cs = w->cs.as<uint32_t>() + b * w->ncs;
        A.qb[b].cap = g->n + 1;
        A.qb[b].ncs = w->ncs;
    }
    A.ctl = w->ctl.as<Ctl>();
    A.rows = reinterpret_cast<hbfs_layer_row *>(w->ctl.as<char>() + sizeof(Ctl));
    A.rows_cap = kRowsCap;
    A.phase_ns = w->phases.as<unsigned long long>();
    A.H.heuristic = p->heuristic;
    A.H.counter_mode = p->counter_mode;
    A.H.force = p->force_direction;
    A.H.alpha = p->alpha;
    A.H.beta = p->beta;
    A.H.n = g->n;
    A.max_pos = p->max_pos;
    A.use_simd = p->use_simd;
    A.parent_mode = p->parent_mode;
    A.root = root;

    int64_t total = 0;
    const Ctl *hc = static_cast<const Ctl *>(w->h_ctl);
    const hbfs_layer_row *hrows =
        reinterpret_cast<const hbfs_layer_row *>(static_cast<const char *>(w->h_ctl) + sizeof(Ctl));
    auto copy_out = [&]() -> int {
        if (parent)
            HB_CUDA(cudaMemcpyAsync(parent, A.parent, g->n * 4, cudaMemcpyDeviceToHost, st));
        if (level)
            HB_CUDA(cudaMemcpyAsync(level, A.level, g->n * 4, cudaMemcpyDeviceToHost, st));
        return HBFS_OK;
    };
    int launches = 0;
    HB_CUDA(cudaEventRecord(w->ev0, st));
    for (int launch = 0;; ++launch) {
        ++launches;
        A.do_init = launch == 0;
        void *kargs[] = {&A};
        HB_CUDA(cudaLaunchCooperativeKernel(w->fn, dim3(w->grid),
                                            dim3(kBlock), kargs, w->smem, st));
        // no-op unless this launch finished the traversal; skipped when the
        // caller asked for parents only (hybrid_bfs: the reference's BfsTree)
        if (!A.direct_levels && level) {
            const int64_t tiles = (g->nw + 31) / 32;
            const int64_t per = kLvBlock / 32;
            const int64_t blocks = std::min<int64_t>((tiles + per - 1) / per, (int64_t)w->lv_grid);
            levels_kernel<OffT><<<(unsigned)std::max<int64_t>(1, blocks), kLvBlock, 0, st>>>(A);
            HB_CUDA(cudaGetLastError());
        }
        HB_CUDA(cudaEventRecord(w->ev1, st));
        // Ctl plus the first rows in one copy; the rest only if needed.
        const size_t head = sizeof(Ctl) + 64 * sizeof(hbfs_layer_row);
        HB_CUDA(cudaMemcpyAsync(w->h_ctl, A.ctl, head, cudaMemcpyDeviceToHost, st));
        // host outputs: queue their copies behind the first launch, so a
        // traversal that finishes in it (all but > kRowsCap layers) costs one
        // stream synchronisation; a resumed traversal copies again at the end
        if (!dev_out && launch == 0) {
            const int rc = copy_out();
            if (rc) return rc;
        }
        HB_CUDA(cudaStreamSynchronize(st));
        const int64_t rows = hc->rows;
        if (rows > 64) {
            HB_CUDA(cudaMemcpyAsync(static_cast<char *>(w->h_ctl) + head,
                                    reinterpret_cast<char *>(A.ctl) + head,
                                    (rows - 64) * sizeof(hbfs_layer_row), cudaMemcpyDeviceToHost, st));
            HB_CUDA(cudaStreamSynchronize(st));
        }
        if (trace) {
            for (int64_t i = 0; i < rows && total + i < trace_cap; ++i) trace[total + i] = hrows[i];
        }
        total += rows;
        if (hc->done) break;  // else: > kRowsCap layers, resume from the persisted state
    }
    if (n_layers) *n_layers = total;
    if (!dev_out && launches > 1) {
        const int rc = copy_out();
        if (rc) return rc;
        HB_CUDA(cudaStreamSynchronize(st));
    }
    if (device_ms) HB_CUDA(cudaEventElapsedTime(device_ms, w->ev0, w->ev1));
    return HBFS_OK;
}

// ------------------------------------------- partition traversal (PART)

// One rank's share of a 1D partition, traversed one layer per launch of the
// persistent kernel (bfs_kernel<..., PART = true>); the host loop and the
// exchange between launches are in csrc/part.cu.
struct PartTrav {
    int64_t n = 0, nw = 0, lo = 0, nown = 0, ncs = 0;
    int cb_ranges = 0, grid = 0;
    size_t smem = 0;
    DevBuf bits, q, qo, qr, cs, cbq, cbqo, cbqr, cbcs, ctl, phases;
    Args<uint64_t> A;
};

static const void *part_kernel() { return (const void *)bfs_kernel<uint64_t, 2, 2, true, true>; }

void *part_trav_create(int64_t n, int64_t lo, int64_t nown, int64_t arcs_local, const uint64_t *rs_local,
                       const uint32_t *adj, const uint32_t *posw_local, const uint4 *hd_local,
                       int64_t n_pos_local, const uint32_t *pre_local, uint32_t *parent_local,
                       int32_t *level_local, uint32_t *cand, uint32_t *touch, int *rc_out, int64_t nw_pad) {
    PartTrav *T = new PartTrav();
    // planes padded to world * (words per rank): the in-place all-gather of a
    // plane writes exactly that many words
    const int64_t nw = std::max<int64_t>((n + 31) / 32, nw_pad);
    T->n = n;
    T->nw = nw;
    T->lo = lo;
    T->nown = nown;
    T->ncs = arcs_local / kTdChunk + 2;
    int rc = T->bits.alloc((1 + kPlanes) * nw * 4 + 64);
    if (!rc) rc = T->q.alloc(2 * (nown + 1) * 4 + 16);
    if (!rc) rc = T->qo.alloc(2 * (nown + 1) * 8);
    if (!rc) rc = T->qr.alloc(2 * (nown + 1) * 8);
    if (!rc) rc = T->cs.alloc(2 * T->ncs * 4);
    T->cb_ranges = n >= env_i64("HBFS_CB_MIN_N", kCbMinN) ? (int)std::min<int64_t>(kCbDefaultRanges, std::max<int64_t>(2, n >> 24)) : 0;
    if (!rc && T->cb_ranges) {
        const int64_t P = T->cb_ranges;
        rc = T->cbq.alloc(P * kCbMaxF * 4);
        if (!rc) rc = T->cbqo.alloc(P * kCbMaxF * 8);
        if (!rc) rc = T->cbqr.alloc(P * kCbMaxF * 8);
        if (!rc) rc = T->cbcs.alloc(P * T->ncs * 4);
    }
    if (!rc) rc = T->ctl.alloc(ctl_bytes());
    if (!rc) rc = T->phases.alloc((kRowsCap + 1) * kPhaseSlots * 8);
    if (!rc) {
        int per_sm = 0, sms = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        T->smem = dyn_smem_bytes<uint64_t>();
        cudaError_t e = cudaFuncSetAttribute(part_kernel(), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T->smem);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, part_kernel(), kBlock, T->smem);
        if (e != cudaSuccess || per_sm < 1) rc = set_error(HBFS_ECUDA, "occupancy query failed");
        T->grid = per_sm * sms;
    }
    if (rc) {
        delete T;
        *rc_out = rc;
        return nullptr;
    }
    Args<uint64_t> &A = T->A;
    memset(&A, 0, sizeof(A));
    // vertex- and word-indexed arrays as offset views: global ids index them
    A.rs = rs_local - lo;
    A.adj = adj;
    A.posw = posw_local - (lo >> 5);
    A.hd = hd_local;  // rank order within the partition
    A.hd2 = hd_local + head2_offset(n_pos_local);
    A.pre = pre_local - (lo >> 5);
    A.n = n;
    A.nw = nw;
    A.arcs = arcs_local;
    A.ncs = T->ncs;
    A.parent = parent_local - lo;
    A.level = level_local - lo;
    A.bits = T->bits.as<uint32_t>();
    for (int b = 0; b < 2; ++b) {
        A.qb[b].q = T->q.as<uint32_t>() + b * (nown + 1);
        A.qb[b].qo = T->qo.as<uint64_t>() + b * (nown + 1);
        A.qb[b].qr = T->qr.as<uint64_t>() + b * (nown + 1);
        A.qb[b].cs = T->cs.as<uint32_t>() + b * T->ncs;
        A.qb[b].cap = nown + 1;
        A.qb[b].ncs = T->ncs;
    }
    A.cbq.q = T->cbq.as<uint32_t>();
    A.cbq.qo = T->cbqo.as<uint64_t>();
    A.cbq.qr = T->cbqr.as<uint64_t>();
    A.cbq.cs = T->cbcs.as<uint32_t>();
    A.cb_ranges = T->cb_ranges;
    A.cb_range_len = T->cb_ranges ? (n + T->cb_ranges - 1) / T->cb_ranges : 0;
    A.cb_cs_stride = T->ncs;
    A.cb_min_arcs = env_i64("HBFS_CB_MIN_ARCS", kCbMinArcs);
    A.harvest_min_arcs = env_i64("HBFS_HARVEST_MIN_ARCS", kHarvestMinArcs);
    A.parent_harvest_min_arcs = env_i64("HBFS_PARENT_HARVEST_MIN_ARCS", kParentHarvestMinArcs);
    // as on one GPU: large graphs record depths in the plane ring and stamp the
    // owned levels once at the end (part_trav_levels)
    A.direct_levels = n < env_i64("HBFS_DEFER_LEVELS_MIN_N", int64_t(1) << 22);
    A.lv_w0 = lo >> 5;
    A.lv_wend = (lo >> 5) + (nown + 31) / 32;
    A.lv_layers = -1;
    A.ctl = T->ctl.as<Ctl>();
    A.rows = reinterpret_cast<hbfs_layer_row *>(T->ctl.as<char>() + sizeof(Ctl));
    A.rows_cap = 1;
    A.phase_ns = T->phases.as<unsigned long long>();
    A.part_w0 = lo >> 5;
    A.part_wend = (lo >> 5) + (nown + 31) / 32;
    A.part_lo = lo;
    A.part_nown = nown;
    A.cand = cand;
    A.touch = touch;
    *rc_out = HBFS_OK;
    return T;
}

void part_trav_free(void *h) { delete static_cast<PartTrav *>(h); }

uint32_t *part_trav_plane(void *h, int64_t depth) {
    PartTrav *T = static_cast<PartTrav *>(h);
    return depth < 0 ? T->bits.as<uint32_t>() : T->bits.as<uint32_t>() + T->nw * (1 + depth % kPlanes);
}

// After the last layer: stamp the owned levels from the depth planes (no-op
// when levels were stamped at discovery).  nL: layers of the traversal.
int part_trav_levels(void *h, int64_t nL, cudaStream_t st) {
    PartTrav *T = static_cast<PartTrav *>(h);
    if (T->A.direct_levels) return HBFS_OK;
    Args<uint64_t> A = T->A;
    A.lv_layers = nL;
    static int lv_grid = 0;
    if (!lv_grid) {
        int per_sm = 0, sms = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, levels_kernel<uint64_t>, kLvBlock, 0);
        lv_grid = std::max(1, per_sm) * sms;
    }
    const int64_t tiles = (A.lv_wend - A.lv_w0 + 31) / 32, per = kLvBlock / 32;
    const int64_t blocks = std::min<int64_t>((tiles + per - 1) / per, (int64_t)lv_grid);
    levels_kernel<uint64_t><<<(unsigned)std::max<int64_t>(1, blocks), kLvBlock, 0, st>>>(A);
    HB_CUDA(cudaGetLastError());
    return HBFS_OK;
}

// One layer, asynchronous: the global controller state in; this rank's
// counters stay on the device — part_trav_add_counters folds them into the
// layer's totals ({found, their degree sum, gathers, fallbacks}) on the
// stream; direction = decide(state).
__global__ void k_add_layer_counters(const Ctr *c, const unsigned long long *applied, unsigned long long *tot) {
    atomicAdd(&tot[0], (c->packed >> kPackShift) + (applied ? applied[0] : 0ull));
    atomicAdd(&tot[1], (c->packed & kPackMask) + (applied ? applied[1] : 0ull));
    atomicAdd(&tot[2], c->gathers);
    atomicAdd(&tot[3], c->fallbacks);
}

int part_trav_add_counters(void *h, int64_t layer, const unsigned long long *applied, unsigned long long *tot,
                           cudaStream_t st) {
    PartTrav *T = static_cast<PartTrav *>(h);
    k_add_layer_counters<<<1, 1, 0, st>>>(&T->A.ctl->ctr[layer % 3], applied, tot);
    HB_CUDA(cudaGetLastError());
    return HBFS_OK;
}

int part_trav_layer(void *h, const int64_t state[6], int32_t dir, int do_init, uint32_t root,
                    const hbfs_params *p, int64_t n_pos_global, unsigned long long *lay_out, int single,
                    cudaStream_t st) {
    PartTrav *T = static_cast<PartTrav *>(h);
    Args<uint64_t> A = T->A;
    A.H.heuristic = p->heuristic;
    A.H.counter_mode = p->counter_mode;
    A.H.force = p->force_direction;
    A.H.alpha = p->alpha;
    A.H.beta = p->beta;
    A.H.n = T->n;
    A.max_pos = p->max_pos;
    A.use_simd = p->use_simd;
    A.parent_mode = HBFS_PARENT_MINID;
    A.root = root;
    A.do_init = do_init;
    A.n_pos = n_pos_global;
    A.bu_exec_ratio = bu_exec_ratio();
    // the controller state travels in the kernel arguments: no copy per layer
    for (int i = 0; i < 6; ++i) A.pst[i] = state[i];
    A.pdir = dir;
    A.part_single = single;
    A.lay_out = lay_out;
    void *kargs[] = {&A};
    HB_CUDA(cudaLaunchCooperativeKernel(part_kernel(), dim3(T->grid), dim3(kBlock), kargs, T->smem, st));
    return HBFS_OK;
}

}  // namespace hbfs

hbfs_graph::~hbfs_graph() { delete ws; }

extern "C" int hbfs_bfs(hbfs_graph *g, int64_t root, const hbfs_params *p, uint32_t *parent,
                        int32_t *level, int on_device, hbfs_layer_row *trace, int64_t trace_cap,
                        int64_t *n_layers, float *device_ms, void *stream) {
    HB_ENTRY_BEGIN
    using namespace hbfs;
    clear_error();
    if (!g || !p) return set_error(HBFS_EINVAL, "null graph or params");
    if (root < 0 || root >= g->n)
        return set_error(HBFS_ERANGE, "source %lld out of range [0, %lld)", (long long)root,
                         (long long)g->n);
    if (p->alpha < 1 || p->beta < 1) return set_error(HBFS_EINVAL, "alpha and beta must be >= 1");
    if (p->max_pos < 1) return set_error(HBFS_EINVAL, "max_pos must be >= 1");
    if (p->force_direction < -1 || p->force_direction > 1)
        return set_error(HBFS_EINVAL, "bad force_direction");
    if (g->n >= (int64_t(1) << 29))
        return set_error(HBFS_ECAPACITY, "single-GPU traversal supports n < 2^29");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lock(g->mu);  // one traversal per graph workspace at a time
    if (g->wide)
        return run_bfs<uint64_t>(g, (uint32_t)root, p, parent, level, on_device, trace, trace_cap,
                                 n_layers, device_ms, st);
    return run_bfs<uint32_t>(g, (uint32_t)root, p, parent, level, on_device, trace, trace_cap,
                             n_layers, device_ms, st);
    HB_ENTRY_END
}

// Diagnostics: per-layer barrier timestamps (ns, device globaltimer) of the last
// launch of the last traversal: slot 0 layer start, 1 after the bitmap->queue
// conversion, 2 after the top-down prologue barrier, 3 after the expansion
// (harvest layers), 4 layer end; 0 = phase not taken.
extern "C" int hbfs_phase_times(hbfs_graph *g, uint64_t *out, int64_t rows) {
    HB_ENTRY_BEGIN
    using namespace hbfs;
    if (!g || !out || rows < 0) return set_error(HBFS_EINVAL, "bad arguments");
    std::lock_guard<std::mutex> lock(g->mu);
    if (!g->ws) return set_error(HBFS_EINVAL, "no traversal yet");
    if (rows > kRowsCap + 1) rows = kRowsCap + 1;
    HB_CUDA(cudaMemcpy(out, g->ws->phases.p, rows * kPhaseSlots * 8, cudaMemcpyDeviceToHost));
    return HBFS_OK;
    HB_ENTRY_END
}

// Device-side index-check flags of a -DHBFS_CHECKED build (bit per check
// site of the traversal kernels, see HB_DCHECK and the bit legend at Ctr);
// *is_checked_build = 0 and *flags = 0 otherwise.
extern "C" int hbfs_debug_checks(uint32_t *flags, int reset, int *is_checked_build) {
    HB_ENTRY_BEGIN
    using namespace hbfs;
    clear_error();
#ifdef HBFS_CHECKED
    if (is_checked_build) *is_checked_build = 1;
    unsigned int f = 0;
    HB_CUDA(cudaDeviceSynchronize());
    HB_CUDA(cudaMemcpyFromSymbol(&f, g_check_fail, sizeof f));
    if (flags) *flags = f;
    if (reset) {
        const unsigned int z = 0;
        HB_CUDA(cudaMemcpyToSymbol(g_check_fail, &z, sizeof z));
    }
#else
    (void)reset;
    if (is_checked_build) *is_checked_build = 0;
    if (flags) *flags = 0;
#endif
    return HBFS_OK;
    HB_ENTRY_END
}
