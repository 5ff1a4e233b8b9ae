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
//   rs     OffT[n+1]   row starts (uint32 when arcs < 2^32, else uint64)
//   adj    u32[arcs]   sorted rows (csr.py:61-64)
//   posw   u32[W]      deg>0 bitmap (engine.py:29-57 `posw`)
//   parent u32[n], level i32[n]
//   bits   u32[4W]     vis | bm0 | bm1 | bm2  — LSB-first bitmaps (frontier.py:3-6)
//   q      u32[2n]     frontier queues (double-buffered)
//   qo     OffT[2(n+1)] exclusive degree prefix of the queue (arc offsets)
//
// Invariants at the start of layer L (depth d = L):
//   in  = bm[L%3] = vertices at depth d (bitmap always valid)
//   visited-before-layer = vis | in          (vis may lag by the frontier)
//   out = bm[(L+1)%3] is all-zero; spare = bm[(L+2)%3] is cleared during L
//   q[L%2]/qo[L%2] valid iff kind == 0 (frontier produced by a top-down layer)
// Parents follow the reference's rule: the minimum-id neighbour one
// level up — TD by atomicMin over all claimers, BU by first hit in the sorted
// row (scans in ascending position order).
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace hbfs {

constexpr int kTdItems = 4;
constexpr int kTdChunk = kBlock * kTdItems;  // arcs per CTA work item
constexpr int kLaneVecs = 2;                 // uint4 probes per lane before the warp scan
constexpr int kPackShift = 35;               // packed counter: count<<35 | degree sum
constexpr unsigned long long kPackMask = (1ull << kPackShift) - 1;
constexpr int64_t kRowsCap = 1024;           // trace rows per launch

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
    int32_t dir, kind, done, pad0;
    int64_t rows;               // rows written by the last launch
    unsigned long long conv;    // enqueue counter of the bitmap->queue phase
    Ctr ctr[3];
};

struct Heur {
    int heuristic, counter_mode, force;
    int64_t alpha, beta, n;
};

// hybrid.py:62-80 (reference rule) / Beamer-GAP rule.  Host+device so the
// controller is identical wherever it runs.
__host__ __device__ inline int decide(const Heur &H, int cur, int64_t v_f, int64_t e_f,
                                      int64_t eu_v, int64_t eu_e, int64_t prev_vf,
                                      int64_t *fv, int64_t *gv) {
    *gv = H.n / H.beta;
    if (H.heuristic == HBFS_HEURISTIC_BEAMER) {
        *fv = eu_e / H.alpha;
        if (H.force >= 0) return H.force;
        if (cur == HBFS_TOP_DOWN) return e_f > *fv ? HBFS_BOTTOM_UP : HBFS_TOP_DOWN;
        return (v_f < prev_vf && v_f <= *gv) ? HBFS_TOP_DOWN : HBFS_BOTTOM_UP;
    }
    const int64_t e_u = H.counter_mode ? eu_e : eu_v;
    *fv = e_u / H.alpha;
    if (H.force >= 0) return H.force;
    if (v_f > *fv) return HBFS_BOTTOM_UP;
    if (v_f < *gv) return HBFS_TOP_DOWN;
    return cur;
}

template <typename OffT>
struct Args {
    const OffT *rs;
    const uint32_t *adj;
    const uint32_t *posw;
    int64_t n, nw, arcs;
    uint32_t *parent;
    int32_t *level;
    uint32_t *bits;  // vis | bm0 | bm1 | bm2
    uint32_t *q;
    OffT *qo;
    Ctl *ctl;
    hbfs_layer_row *rows;
    int64_t rows_cap;
    Heur H;
    int max_pos, use_simd, parent_mode, do_init;
    uint32_t root;
};

struct St {
    int64_t layer, v_f, e_f, eu_v, eu_e, prev_vf;
    int dir, kind;
};

template <typename OffT>
struct TdSmem {
    OffT off[kTdChunk + 2];
    OffT rs[kTdChunk + 2];
    uint32_t u[kTdChunk + 2];
    int64_t q0, cnt;
};

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Largest index j in [0, len) with a[j] <= x (a non-decreasing, a[0] <= x).
template <typename OffT>
__device__ __forceinline__ int64_t last_le(const OffT *a, int64_t len, uint64_t x) {
    int64_t lo = 0, hi = len;  // invariant: a[lo] <= x, answer in [lo, hi)
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if ((uint64_t)a[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

// Warp-aggregated append of (v, deg) into a queue with its arc-offset prefix:
// one 64-bit atomic per warp reserves both the slots and the arc range, so
// queue order and prefix order agree (count<<35 | degree sum).
template <typename OffT>
__device__ __forceinline__ void warp_enqueue(bool claim, uint32_t v, uint64_t deg,
                                             unsigned long long *counter, uint32_t *NQ,
                                             OffT *NQO) {
    const unsigned full = 0xffffffffu;
    const unsigned m = __ballot_sync(full, claim);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    uint64_t x = claim ? deg : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(full, x, o);
        if (lane >= o) x += y;
    }
    const uint64_t total = __shfl_sync(full, x, 31);
    const uint64_t excl = x - (claim ? deg : 0);
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (lane == leader)
        base = atomicAdd(counter, ((unsigned long long)__popc(m) << kPackShift) + total);
    base = __shfl_sync(full, base, leader);
    if (claim) {
        const uint64_t pos = (base >> kPackShift) + __popc(m & ((1u << lane) - 1));
        NQ[pos] = v;
        NQO[pos] = (OffT)((base & kPackMask) + excl);
    }
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    return x;
}

// ---------------------------------------------------------------- phases

template <typename OffT>
__device__ void phase_init(const Args<OffT> &A) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const uint32_t root = A.root;
    for (int64_t i = tid; i < A.n; i += nth) {
        const bool r = i == (int64_t)root;
        A.parent[i] = r ? root : HBFS_NIL;
        A.level[i] = r ? 0 : -1;
    }
    const int64_t rootw = A.nw + (root >> 5);  // bm0 word holding the root
    for (int64_t w = tid; w < 4 * A.nw; w += nth)
        A.bits[w] = (w == rootw) ? (1u << (root & 31)) : 0u;
    if (tid == 0) {
        A.q[0] = root;
        A.qo[0] = 0;
        Ctl *c = A.ctl;
        for (int s = 0; s < 3; ++s) c->ctr[s] = Ctr{0, 0, 0, 0};
        c->conv = 0;
        c->done = 0;
    }
}

// Top-down layer: arc-balanced expansion of the frontier queue.  CTA work item =
// kTdChunk consecutive arcs of the concatenated frontier rows (so hubs of any
// degree spread over many CTAs and adjacency reads are coalesced); each thread
// maps its arc to (u, position) by binary search in the CTA's slice of the
// degree prefix.  Replaces top_down_layer/top_down_chunked (_native.pyx:65-86,
// :207-239).
template <typename OffT>
__device__ void phase_td(const Args<OffT> &A, const St &S, const uint32_t *in, uint32_t *out,
                         uint32_t *spare, Ctr *ctr, TdSmem<OffT> &sm) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t cur = S.layer & 1;
    const uint32_t *Q = A.q + cur * A.n;
    const OffT *QO = A.qo + cur * (A.n + 1);
    uint32_t *NQ = A.q + (1 - cur) * A.n;
    OffT *NQO = A.qo + (1 - cur) * (A.n + 1);
    uint32_t *vis = A.bits;
    const int64_t nf = S.v_f;
    const uint64_t mf = (uint64_t)S.e_f;
    const int32_t depth1 = (int32_t)S.layer + 1;

    for (int64_t i = tid; i < nf; i += nth) {  // commit the frontier to vis
        const uint32_t u = Q[i];
        atomicOr(&vis[u >> 5], 1u << (u & 31));
    }
    for (int64_t w = tid; w < A.nw; w += nth) spare[w] = 0;

    const int64_t nchunks = (int64_t)((mf + kTdChunk - 1) / kTdChunk);
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const uint64_t a0 = (uint64_t)c * kTdChunk;
        const uint64_t a1 = min(a0 + (uint64_t)kTdChunk, mf);
        if (threadIdx.x == 0) {
            const int64_t q0 = last_le(QO, nf, a0);
            const int64_t q1 = last_le(QO, nf, a1 - 1);
            sm.q0 = q0;
            sm.cnt = q1 - q0 + 1;
        }
        __syncthreads();
        const int64_t q0 = sm.q0, cnt = sm.cnt;
        const bool in_smem = cnt <= kTdChunk + 2;
        if (in_smem) {
            for (int64_t j = threadIdx.x; j < cnt; j += blockDim.x) {
                const uint32_t u = Q[q0 + j];
                sm.u[j] = u;
                sm.off[j] = QO[q0 + j];
                sm.rs[j] = __ldg(A.rs + u);
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kTdItems; ++k) {
            const uint64_t a = a0 + (uint64_t)k * blockDim.x + threadIdx.x;
            bool claim = false;
            uint32_t v = 0;
            uint64_t deg = 0;
            if (a < a1) {
                uint32_t u;
                OffT off, rsu;
                if (in_smem) {
                    const int64_t j = last_le(sm.off, cnt, a);
                    off = sm.off[j];
                    u = sm.u[j];
                    rsu = sm.rs[j];
                } else {
                    const int64_t j = q0 + last_le(QO + q0, nf - q0, a);
                    off = QO[j];
                    u = Q[j];
                    rsu = __ldg(A.rs + u);
                }
                v = __ldg(A.adj + (uint64_t)rsu + (a - (uint64_t)off));
                const uint32_t w = v >> 5, b = 1u << (v & 31);
                const uint32_t seen = vis[w] | in[w];
                if (!(seen & b)) {
                    uint32_t old = out[w];
                    if (!(old & b)) old = atomicOr(&out[w], b);
                    claim = !(old & b);
                    if (A.parent_mode == HBFS_PARENT_MINID) atomicMin(&A.parent[v], u);
                    else if (claim) A.parent[v] = u;
                    if (claim) {
                        A.level[v] = depth1;
                        deg = (uint64_t)(__ldg(A.rs + v + 1) - __ldg(A.rs + v));
                    }
                }
            }
            warp_enqueue(claim, v, deg, &ctr->packed, NQ, NQO);
        }
        __syncthreads();
    }
}

// Bottom-up layer: one warp per 32-vertex bitmap word (the warp owns the word,
// so vis/out updates are plain stores).  Each lane probes its own sorted row in
// ascending position with aligned uint4 loads; lanes still unresolved after
// kLaneVecs vectors hand their remaining row to a warp-cooperative scan that
// takes the lowest hit position (ballot + ffs), preserving the reference's
// first-hit rule.  Counters gathers/fallbacks are those the reference's
// 16-lane kernel would report.  Replaces bottom_up_multiple_set /
// bottom_up_layer (_native.pyx:89-204, bu_probe.h:22-106).
template <typename OffT>
__device__ void phase_bu(const Args<OffT> &A, const St &S, const uint32_t *in, uint32_t *out,
                         uint32_t *spare, Ctr *ctr, unsigned long long *red) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = tid >> 5, nwarps = nth >> 5;
    uint32_t *vis = A.bits;
    const int32_t depth1 = (int32_t)S.layer + 1;
    const int64_t max_pos = A.max_pos;
    unsigned long long c_cnt = 0, c_deg = 0, c_gat = 0, c_fb = 0;

    for (int64_t w = tid; w < A.nw; w += nth) spare[w] = 0;

    for (int64_t w = gwarp; w < A.nw; w += nwarps) {
        const uint32_t vw = vis[w], iw = in[w], pw = __ldg(A.posw + w);
        const uint32_t visited = vw | iw;
        const uint32_t cand = ~visited & pw;
        if (!cand) {
            if (lane == 0 && iw && (vw | iw) != vw) vis[w] = visited;
            continue;
        }
        const bool mine = (cand >> lane) & 1u;
        const uint64_t v = (uint64_t)w * 32 + lane;
        OffT s = 0, e = 0;
        if (mine) {
            s = __ldg(A.rs + v);
            e = __ldg(A.rs + v + 1);
        }
        int64_t hit = -1;  // absolute adjacency index of the first frontier neighbour
        uint32_t hit_u = 0;
        OffT p = s;
        if (mine) {
#pragma unroll
            for (int it = 0; it < kLaneVecs; ++it) {
                if (p >= e) break;
                const OffT base = p & ~(OffT)3;
                const uint4 q4 = __ldg(reinterpret_cast<const uint4 *>(A.adj + base));
                const uint32_t val[4] = {q4.x, q4.y, q4.z, q4.w};
                uint32_t hm = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const OffT idx = base + j;
                    if (idx >= p && idx < e) {
                        const uint32_t a = val[j];
                        if ((in[a >> 5] >> (a & 31)) & 1u) hm |= 1u << j;
                    }
                }
                if (hm) {
                    const int j = __ffs(hm) - 1;
                    hit = (int64_t)(base + j);
                    hit_u = val[j];
                    break;
                }
                p = base + 4;
            }
        }
        unsigned todo = __ballot_sync(0xffffffffu, mine && hit < 0 && p < e);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint64_t ps = (uint64_t)__shfl_sync(0xffffffffu, (unsigned long long)p, src);
            const uint64_t pe = (uint64_t)__shfl_sync(0xffffffffu, (unsigned long long)e, src);
            int64_t h = -1;
            uint32_t hu = 0;
            for (uint64_t c = ps; c < pe; c += 32) {
                const uint64_t idx = c + lane;
                bool bit = false;
                uint32_t a = 0;
                if (idx < pe) {
                    a = __ldg(A.adj + idx);
                    bit = (in[a >> 5] >> (a & 31)) & 1u;
                }
                const unsigned hb = __ballot_sync(0xffffffffu, bit);
                if (hb) {
                    const int l = __ffs(hb) - 1;
                    h = (int64_t)(c + l);
                    hu = __shfl_sync(0xffffffffu, a, l);
                    break;
                }
            }
            if (lane == src && h >= 0) {
                hit = h;
                hit_u = hu;
            }
        }
        const bool found = hit >= 0;
        if (found) {
            A.parent[v] = hit_u;
            A.level[v] = depth1;
        }
        const unsigned fm = __ballot_sync(0xffffffffu, found);
        if (lane == 0) {
            if (fm) out[w] = fm;
            if ((iw | fm) && (visited | fm) != vw) vis[w] = visited | fm;
        }
        if (mine) {
            const int64_t deg = (int64_t)(e - s);
            const int64_t pos = found ? hit - (int64_t)s : -1;
            const bool early = found && pos < max_pos;
            if (found) {
                c_cnt += 1;
                c_deg += (unsigned long long)deg;
            }
            c_gat += early ? (unsigned long long)(pos + 1)
                           : (unsigned long long)(deg < max_pos ? deg : max_pos);
            c_fb += (deg > max_pos && !early) ? 1ull : 0ull;
        }
    }
    // CTA reduction of the counters, one atomic per CTA per counter.
    c_cnt = warp_sum(c_cnt);
    c_deg = warp_sum(c_deg);
    c_gat = warp_sum(c_gat);
    c_fb = warp_sum(c_fb);
    const int wid = threadIdx.x >> 5;
    if (lane == 0) {
        red[wid * 4 + 0] = c_cnt;
        red[wid * 4 + 1] = c_deg;
        red[wid * 4 + 2] = c_gat;
        red[wid * 4 + 3] = c_fb;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t[4] = {0, 0, 0, 0};
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i)
            for (int k = 0; k < 4; ++k) t[k] += red[i * 4 + k];
        if (t[0] | t[1]) atomicAdd(&ctr->packed, (t[0] << kPackShift) + t[1]);
        if (t[2]) atomicAdd(&ctr->gathers, t[2]);
        if (t[3]) atomicAdd(&ctr->fallbacks, t[3]);
    }
    __syncthreads();
}

// Bitmap -> queue (with arc-offset prefix) at a bottom-up -> top-down switch.
template <typename OffT>
__device__ void phase_convert(const Args<OffT> &A, const St &S, const uint32_t *in) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const int64_t cur = S.layer & 1;
    uint32_t *Q = A.q + cur * A.n;
    OffT *QO = A.qo + cur * (A.n + 1);
    for (int64_t w0 = tid - lane; w0 < A.nw; w0 += nth) {
        const int64_t w = w0 + lane;
        uint32_t bits = w < A.nw ? in[w] : 0u;
        while (__any_sync(0xffffffffu, bits != 0)) {
            const bool has = bits != 0;
            uint32_t v = 0;
            uint64_t deg = 0;
            if (has) {
                v = (uint32_t)(w * 32 + __ffs(bits) - 1);
                bits &= bits - 1;
                deg = (uint64_t)(__ldg(A.rs + v + 1) - __ldg(A.rs + v));
            }
            warp_enqueue(has, v, deg, &A.ctl->conv, Q, QO);
        }
    }
}

template <typename OffT>
__global__ void __launch_bounds__(kBlock) bfs_kernel(Args<OffT> A) {
    cg::grid_group grid = cg::this_grid();
    __shared__ TdSmem<OffT> sm;
    __shared__ unsigned long long red[(kBlock / 32) * 4];
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;

    St S;
    if (A.do_init) {
        phase_init(A);
        grid.sync();
        const int64_t rdeg = (int64_t)(__ldg(A.rs + A.root + 1) - __ldg(A.rs + A.root));
        S.layer = 0;
        S.v_f = 1;
        S.e_f = rdeg;
        S.eu_v = A.n - 1;
        S.eu_e = A.arcs - rdeg;
        S.prev_vf = 0;
        S.dir = HBFS_TOP_DOWN;
        S.kind = 0;
    } else {
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
    while (S.v_f > 0 && rows < A.rows_cap) {
        int64_t fv, gv;
        const int dir = decide(A.H, S.dir, S.v_f, S.e_f, S.eu_v, S.eu_e, S.prev_vf, &fv, &gv);
        const int64_t L = S.layer;
        const uint32_t *in = A.bits + A.nw * (1 + L % 3);
        uint32_t *out = A.bits + A.nw * (1 + (L + 1) % 3);
        uint32_t *spare = A.bits + A.nw * (1 + (L + 2) % 3);
        Ctr *ctr = &A.ctl->ctr[L % 3];
        if (dir == HBFS_TOP_DOWN && S.kind == 1) {
            phase_convert(A, S, in);
            grid.sync();
        }
        // Slot (L+1)%3 was last read right after the barrier that ended layer
        // L-2, so every CTA is past that read; it must be zero when layer L+1
        // starts accumulating.  The conversion counter is free again too.
        if (leader) {
            A.ctl->ctr[(L + 1) % 3] = Ctr{0, 0, 0, 0};
            A.ctl->conv = 0;
        }
        if (dir == HBFS_TOP_DOWN) phase_td(A, S, in, out, spare, ctr, sm);
        else phase_bu(A, S, in, out, spare, ctr, red);
        grid.sync();

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
        }
        S.prev_vf = S.v_f;
        S.v_f = nvf;
        S.e_f = nef;
        S.eu_v -= nvf;
        S.eu_e -= nef;
        S.dir = dir;
        S.kind = dir == HBFS_TOP_DOWN ? 0 : 1;
        S.layer = L + 1;
        ++rows;
    }
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

// ------------------------------------------------------------ workspace

struct Workspace {
    int64_t n = 0;
    int wide = 0;
    DevBuf parent, level, bits, q, qo, ctl;  // ctl: Ctl followed by kRowsCap rows
    int grid = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    void *h_ctl = nullptr;  // pinned mirror of ctl + rows
    ~Workspace() {
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (h_ctl) cudaFreeHost(h_ctl);
    }
};

static size_t ctl_bytes() { return sizeof(Ctl) + kRowsCap * sizeof(hbfs_layer_row); }

template <typename OffT>
static int ws_alloc(hbfs_graph *g) {
    if (g->ws) return HBFS_OK;
    Workspace *w = new Workspace();
    const int64_t n = g->n, nw = g->nw;
    int rc = HBFS_OK;
    if (!rc) rc = w->parent.alloc(n * 4);
    if (!rc) rc = w->level.alloc(n * 4);
    if (!rc) rc = w->bits.alloc(4 * nw * 4 + 16);
    if (!rc) rc = w->q.alloc(2 * n * 4 + 16);
    if (!rc) rc = w->qo.alloc(2 * (n + 1) * sizeof(OffT));
    if (!rc) rc = w->ctl.alloc(ctl_bytes());
    if (!rc && cudaMallocHost(&w->h_ctl, ctl_bytes()) != cudaSuccess)
        rc = set_error(HBFS_ECUDA, "cudaMallocHost failed");
    if (!rc && (cudaEventCreate(&w->ev0) != cudaSuccess || cudaEventCreate(&w->ev1) != cudaSuccess))
        rc = set_error(HBFS_ECUDA, "cudaEventCreate failed");
    if (!rc) {
        int per_sm = 0, sms = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_kernel<OffT>, kBlock, 0);
        if (e != cudaSuccess || per_sm < 1)
            rc = set_error(HBFS_ECUDA, "occupancy query failed: %s", cudaGetErrorString(e));
        w->grid = per_sm * sms;
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
    A.n = g->n;
    A.nw = g->nw;
    A.arcs = g->arcs;
    const bool dev_out = on_device != 0;
    A.parent = (dev_out && parent) ? parent : w->parent.as<uint32_t>();
    A.level = (dev_out && level) ? level : w->level.as<int32_t>();
    A.bits = w->bits.as<uint32_t>();
    A.q = w->q.as<uint32_t>();
    A.qo = w->qo.as<OffT>();
    A.ctl = w->ctl.as<Ctl>();
    A.rows = reinterpret_cast<hbfs_layer_row *>(w->ctl.as<char>() + sizeof(Ctl));
    A.rows_cap = kRowsCap;
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
    HB_CUDA(cudaEventRecord(w->ev0, st));
    for (int launch = 0;; ++launch) {
        A.do_init = launch == 0;
        void *kargs[] = {&A};
        HB_CUDA(cudaLaunchCooperativeKernel((const void *)bfs_kernel<OffT>, dim3(w->grid),
                                            dim3(kBlock), kargs, 0, st));
        HB_CUDA(cudaEventRecord(w->ev1, st));
        // Ctl plus the first rows in one copy; the rest only if needed.
        const size_t head = sizeof(Ctl) + 64 * sizeof(hbfs_layer_row);
        HB_CUDA(cudaMemcpyAsync(w->h_ctl, A.ctl, head, cudaMemcpyDeviceToHost, st));
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
    if (!dev_out) {
        if (parent)
            HB_CUDA(cudaMemcpyAsync(parent, A.parent, g->n * 4, cudaMemcpyDeviceToHost, st));
        if (level)
            HB_CUDA(cudaMemcpyAsync(level, A.level, g->n * 4, cudaMemcpyDeviceToHost, st));
    }
    HB_CUDA(cudaStreamSynchronize(st));
    if (device_ms) HB_CUDA(cudaEventElapsedTime(device_ms, w->ev0, w->ev1));
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
    if (g->wide)
        return run_bfs<uint64_t>(g, (uint32_t)root, p, parent, level, on_device, trace, trace_cap,
                                 n_layers, device_ms, st);
    return run_bfs<uint32_t>(g, (uint32_t)root, p, parent, level, on_device, trace, trace_cap,
                             n_layers, device_ms, st);
    HB_ENTRY_END
}
