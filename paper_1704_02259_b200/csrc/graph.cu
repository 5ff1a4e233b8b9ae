// Graph input on device: R-MAT generator, CSR build, CSR import/export and
// source sampling.  Replaces generator.generate (generator.py:136-159),
// csr.from_arrays (csr.py:46-74) and harness.sample_sources
// (harness.py:73-97).  All of it is integer work and bit-exact with the
// reference: mix64 is a bijection, so every sort key is distinct and any sort
// reproduces numpy's stable argsort / key sort.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace hbfs {

static thread_local std::string g_err;

int set_error(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

void clear_error() { g_err.clear(); }

static inline int grid_for(int64_t items, int block = 256) {
    int64_t g = (items + block - 1) / block;
    if (g > 148 * 64) g = 148 * 64;
    return (int)(g < 1 ? 1 : g);
}

// ------------------------------------------------------------- generator

// One thread per edge: h0 = mix64(e*GOLDEN + seed) once, then `scale` levels of
// h = mix64(h0 ^ (level+1)*SALT), r = (h>>11)*2^-53 (generator.py:47-53).  The
// float64 comparisons r >= t are done exactly in integers: r = k*2^-53 with k an
// integer, so r >= t  <=>  k >= ceil(t*2^53) (host-computed, exact).
__global__ void k_gen_edges(int scale, int64_t m, uint64_t seed, uint64_t ka, uint64_t kab,
                            uint64_t kabc, uint32_t *u, uint32_t *v) {
    const uint64_t golden = 0x9E3779B97F4A7C15ull, salt0 = 0xD6E8FEB86659FD93ull;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h0 = mix64((uint64_t)e * golden + seed);
        uint32_t uu = 0, vv = 0;
        for (int lv = 0; lv < scale; ++lv) {
            const uint64_t k = mix64(h0 ^ ((uint64_t)(lv + 1) * salt0)) >> 11;
            uu = (uu << 1) | (uint32_t)(k >= kab);
            vv = (vv << 1) | (uint32_t)(((k >= ka) && (k < kab)) || (k >= kabc));
        }
        u[e] = uu;
        v[e] = vv;
    }
}

__global__ void k_perm_keys(int64_t n, uint64_t seed, uint64_t add, uint64_t *key, uint32_t *id) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        key[i] = mix64(mix64((uint64_t)i + add) ^ seed);
        id[i] = (uint32_t)i;
    }
}

__global__ void k_apply_perm(int64_t m, const uint32_t *perm, uint32_t *u, uint32_t *v) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        u[e] = perm[u[e]];
        v[e] = perm[v[e]];
    }
}

static uint64_t exact_threshold(double t) {
    // ceil(t * 2^53) for t in [0, 1] (power-of-two scaling is exact).
    double s = std::ldexp(t, 53);
    double c = std::ceil(s);
    if (c < 0) c = 0;
    return (uint64_t)c;
}

// argsort of mix64(mix64(i + add) ^ seed) over i < n  (generator.py:129-133,
// harness.py:85-87).  Result: sorted ids in `out` (device, n entries).
static int keyed_order(int64_t n, uint64_t seed, uint64_t add, uint32_t *out, cudaStream_t st) {
    DevBuf k0, k1, i0, tmp;
    HB_CHECK(k0.alloc(n * 8));
    HB_CHECK(k1.alloc(n * 8));
    HB_CHECK(i0.alloc(n * 4));
    k_perm_keys<<<grid_for(n), 256, 0, st>>>(n, seed, add, k0.as<uint64_t>(), i0.as<uint32_t>());
    HB_CUDA(cudaGetLastError());
    size_t tb = 0;
    HB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0.as<uint64_t>(), k1.as<uint64_t>(),
                                            i0.as<uint32_t>(), out, n, 0, 64, st));
    HB_CHECK(tmp.alloc(tb));
    HB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, k0.as<uint64_t>(), k1.as<uint64_t>(),
                                            i0.as<uint32_t>(), out, n, 0, 64, st));
    return HBFS_OK;
}

static int gen_edges_dev(int scale, int64_t ef, uint64_t seed, const double thr[3], int permute,
                         uint32_t *du, uint32_t *dv, cudaStream_t st) {
    const int64_t n = int64_t(1) << scale;
    const int64_t m = n * ef;
    k_gen_edges<<<grid_for(m), 256, 0, st>>>(scale, m, seed, exact_threshold(thr[0]),
                                             exact_threshold(thr[1]), exact_threshold(thr[2]),
                                             du, dv);
    HB_CUDA(cudaGetLastError());
    if (permute && n > 1) {
        DevBuf perm;
        HB_CHECK(perm.alloc(n * 4));
        HB_CHECK(keyed_order(n, seed, 1, perm.as<uint32_t>(), st));
        k_apply_perm<<<grid_for(m), 256, 0, st>>>(m, perm.as<uint32_t>(), du, dv);
        HB_CUDA(cudaGetLastError());
        HB_CUDA(cudaStreamSynchronize(st));
    }
    return HBFS_OK;
}

// ------------------------------------------------------------------- CSR

static int bits_for(int64_t n) {
    int b = 0;
    while ((int64_t(1) << b) < n) ++b;
    return b < 1 ? 1 : b;
}

// keys for both arc directions: (src << sb) | dst  (csr.py:54-55, :62)
__global__ void k_arc_keys(int64_t m, int sb, const uint32_t *u, const uint32_t *v, uint64_t *key) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t a = u[e], b = v[e];
        key[e] = (a << sb) | b;
        key[m + e] = (b << sb) | a;
    }
}

// dedup flags: keep first of equal keys, drop self-loops
__global__ void k_dedup_flags(int64_t arcs, int sb, const uint64_t *key, uint8_t *keep) {
    const uint64_t mask = (uint64_t(1) << sb) - 1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < arcs;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = key[i];
        const bool self = (k >> sb) == (k & mask);
        const bool dup = i > 0 && key[i - 1] == k;
        keep[i] = !(self || dup);
    }
}

__global__ void k_key_to_adj(int64_t arcs, int sb, const uint64_t *key, uint32_t *adj) {
    const uint64_t mask = (uint64_t(1) << sb) - 1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < arcs;
         i += (int64_t)gridDim.x * blockDim.x)
        adj[i] = (uint32_t)(key[i] & mask);
}

// row_starts[v] = lower_bound(keys, v << sb)  (equivalent to cumsum(bincount))
template <typename OffT>
__global__ void k_row_starts(int64_t n, int64_t arcs, int sb, const uint64_t *key, OffT *rs) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t target = (uint64_t)v << sb;
        int64_t lo = 0, hi = arcs;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (key[mid] < target) lo = mid + 1; else hi = mid;
        }
        rs[v] = (OffT)lo;
    }
}

template <typename OffT>
__global__ void k_posw(int64_t n, int64_t nw, const OffT *rs, uint32_t *posw,
                       unsigned long long *maxdeg) {
    const int lane = threadIdx.x & 31;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t v = w * 32 + lane;
        uint64_t d = 0;
        if (v < n) d = (uint64_t)(rs[v + 1] - rs[v]);
        const unsigned b = __ballot_sync(0xffffffffu, d > 0);
        uint64_t mx = d;
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t y = __shfl_down_sync(0xffffffffu, mx, o);
            mx = y > mx ? y : mx;
        }
        if (lane == 0) {
            posw[w] = b;
            if (mx) atomicMax(maxdeg, (unsigned long long)mx);
        }
    }
}

// Head records (common.cuh), packed in rank order over the vertices with
// degree > 0: pre[w] = number of such vertices before bitmap word w, so vertex
// v = 32 w + b sits at pre[w] + popc(posw[w] & ((1 << b) - 1)).
struct PopcOp {
    __host__ __device__ uint32_t operator()(uint32_t x) const {
#ifdef __CUDA_ARCH__
        return __popc(x);
#else
        return (uint32_t)__builtin_popcount(x);
#endif
    }
};

template <typename OffT>
__global__ void k_heads(int64_t n, const OffT *rs, const uint32_t *adj, const uint32_t *posw,
                        const uint32_t *pre, uint4 *hd, uint4 *hd2) {
    constexpr int RW = sizeof(OffT) / 4;  // words of the row start in the second-tier record
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const OffT s = rs[v];
        const uint64_t d = (uint64_t)(rs[v + 1] - s);
        if (d == 0) continue;
        uint4 h;
        h.x = (uint32_t)d;
        h.y = adj[(uint64_t)s];
        h.z = d > 1 ? adj[(uint64_t)s + 1] : HBFS_NIL;
        h.w = d > 2 ? adj[(uint64_t)s + 2] : HBFS_NIL;
        const int64_t slot = pre[v >> 5] + __popc(posw[v >> 5] & ((1u << (v & 31)) - 1u));
        hd[slot] = h;
        uint32_t w[kH2W];
        w[0] = (uint32_t)((uint64_t)s & 0xFFFFFFFFu);
        if (RW == 2) w[1] = (uint32_t)((uint64_t)s >> 32);
#pragma unroll
        for (int j = RW; j < kH2W; ++j) {
            const uint64_t pos = (uint64_t)kHeadLen + (j - RW);
            w[j] = pos < d ? adj[(uint64_t)s + pos] : HBFS_NIL;
        }
#pragma unroll
        for (int q = 0; q < kH2W / 4; ++q)
            hd2[(kH2W / 4) * slot + q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    }
}

int build_heads(int64_t n, const void *rs, int wide, const uint32_t *adj, const uint32_t *posw,
                DevBuf &pre, DevBuf &hd, cudaStream_t st, int64_t *n_records) {
    static_assert(kHeadLen == 3, "head record layout");
    const int64_t nw = (n + 31) / 32;
    HB_CHECK(pre.alloc((nw + 1) * 4 + 16));
    uint32_t total = 0;
    if (nw > 0) {
        // exclusive scan over nw + 1 items: pre[nw] = number of records (posw
        // is allocated with slack, the value read at nw does not matter)
        cub::TransformInputIterator<uint32_t, PopcOp, const uint32_t *> in(posw, PopcOp());
        size_t tb = 0;
        HB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, pre.as<uint32_t>(), nw + 1, st));
        DevBuf tmp;
        HB_CHECK(tmp.alloc(tb));
        HB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, pre.as<uint32_t>(), nw + 1, st));
        HB_CUDA(cudaMemcpyAsync(&total, pre.as<uint32_t>() + nw, 4, cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaStreamSynchronize(st));
    }
    if (n_records) *n_records = (int64_t)total;
    const int64_t off2 = head2_offset((int64_t)total);
    HB_CHECK(hd.alloc(((size_t)off2 + (kH2W / 4) * ((size_t)total + 1)) * sizeof(uint4)));
    if (n <= 0) return HBFS_OK;
    const int blocks = grid_for(n);
    if (wide)
        k_heads<uint64_t><<<blocks, 256, 0, st>>>(n, static_cast<const uint64_t *>(rs), adj, posw,
                                                 pre.as<uint32_t>(), hd.as<uint4>(), hd.as<uint4>() + off2);
    else
        k_heads<uint32_t><<<blocks, 256, 0, st>>>(n, static_cast<const uint32_t *>(rs), adj, posw,
                                                 pre.as<uint32_t>(), hd.as<uint4>(), hd.as<uint4>() + off2);
    HB_CUDA(cudaGetLastError());
    HB_CUDA(cudaStreamSynchronize(st));
    return HBFS_OK;
}

// Structural check of a caller-supplied CSR (hbfs_graph_from_csr, csr.load of a
// cache blob): bit 0 row_starts[0] != 0, bit 1 row_starts decreases somewhere,
// bit 2 an adjacency id >= n.  The traversal kernels index parent/level/bitmaps
// by adjacency values, so a corrupt CSR must be refused, not traversed.
__global__ void k_check_csr(int64_t n, int64_t arcs, const int64_t *rs, const uint32_t *adj,
                            unsigned *bad) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned f = 0;
    if (t0 == 0 && rs[0] != 0) f |= 1u;
    for (int64_t i = t0; i < n; i += stride)
        if (rs[i + 1] < rs[i]) f |= 2u;
    for (int64_t i = t0; i < arcs; i += stride)
        if ((int64_t)adj[i] >= n) f |= 4u;
    f = __reduce_or_sync(0xffffffffu, f);
    if (f && (threadIdx.x & 31) == 0) atomicOr(bad, f);
}

__global__ void k_narrow(int64_t cnt, const int64_t *src, uint32_t *dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = (uint32_t)src[i];
}

template <typename OffT>
__global__ void k_widen(int64_t cnt, const OffT *src, int64_t *dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = (int64_t)src[i];
}

// posw + max degree.  Called once the rs (OffT) and adj arrays are in place.
int graph_finalize(hbfs_graph *g, cudaStream_t st) {
    g->nw = (g->n + 31) / 32;
    HB_CHECK(g->posw.alloc(g->nw * 4 + 16));
    DevBuf md;
    HB_CHECK(md.alloc(8));
    HB_CUDA(cudaMemsetAsync(md.p, 0, 8, st));
    if (g->nw > 0) {
        const int blocks = grid_for(g->nw * 32);
        if (g->wide)
            k_posw<uint64_t><<<blocks, 256, 0, st>>>(g->n, g->nw, g->rs.as<uint64_t>(),
                                                    g->posw.as<uint32_t>(), md.as<unsigned long long>());
        else
            k_posw<uint32_t><<<blocks, 256, 0, st>>>(g->n, g->nw, g->rs.as<uint32_t>(),
                                                    g->posw.as<uint32_t>(), md.as<unsigned long long>());
        HB_CUDA(cudaGetLastError());
    }
    unsigned long long h = 0;
    HB_CUDA(cudaMemcpyAsync(&h, md.p, 8, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    g->max_degree = (int64_t)h;
    cudaGetDevice(&g->device);
    if (g->max_degree >= (int64_t(1) << 32))
        return set_error(HBFS_ECAPACITY, "a row of %lld entries exceeds the 32-bit degree of the head records",
                         (long long)g->max_degree);
    HB_CHECK(build_heads(g->n, g->rs.p, g->wide, g->adj.as<uint32_t>(), g->posw.as<uint32_t>(), g->pre, g->hd, st, &g->n_pos));
    return HBFS_OK;
}

static int alloc_adj(hbfs_graph *g) {
    // +8 entries: aligned uint4 probes may read up to 3 entries past the end
    HB_CHECK(g->adj.alloc((g->arcs + 8) * 4));
    return HBFS_OK;
}

// ---- source-range build for graphs whose monolithic key sort does not fit
// (SCALE 28: 2^33 arcs = 2 x 69 GB of keys).  The vertex range is cut into P
// pieces; piece r sorts only the arcs whose source lies in it, with keys
// (src - lo) << sb | dst, and writes its rows at the running arc offset.  Rows
// come out in (src, dst) order exactly as in the monolithic build (and
// csr.py:54-64).

// arcs per source piece (both directions of every edge)
__global__ void k_piece_counts(int64_t m, const uint32_t *u, const uint32_t *v, int64_t span, int P,
                               unsigned long long *cnt) {
    extern __shared__ unsigned long long s_cnt[];
    for (int i = threadIdx.x; i < P; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        atomicAdd(&s_cnt[u[e] / span], 1ull);
        atomicAdd(&s_cnt[v[e] / span], 1ull);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < P; i += blockDim.x)
        if (s_cnt[i]) atomicAdd(&cnt[i], s_cnt[i]);
}

// keys of the arcs whose source is in [lo, lo + span); warp-aggregated slots
__global__ void k_piece_keys(int64_t m, const uint32_t *u, const uint32_t *v, int64_t lo, int64_t span,
                             int sb, uint64_t *key, unsigned long long *pos) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t m32 = (m + 31) & ~int64_t(31);  // whole warps iterate together
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m32; e += stride) {
        const bool in = e < m;
        const uint32_t a = in ? u[e] : 0u, b = in ? v[e] : 0u;
        const bool fa = in && (int64_t)a >= lo && (int64_t)a < lo + span;
        const bool fb = in && (int64_t)b >= lo && (int64_t)b < lo + span;
        const unsigned ba = __ballot_sync(0xffffffffu, fa), bb = __ballot_sync(0xffffffffu, fb);
        const unsigned tot = __popc(ba) + __popc(bb);
        if (!tot) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(pos, (unsigned long long)tot);
        base = __shfl_sync(0xffffffffu, base, 0);
        const unsigned below = (1u << lane) - 1u;
        if (fa) key[base + __popc(ba & below)] = ((uint64_t)(a - lo) << sb) | b;
        if (fb) key[base + __popc(ba) + __popc(bb & below)] = ((uint64_t)(b - lo) << sb) | a;
    }
}

// rs[lo + i] = off + lower_bound(keys, i << sb) for local rows i in [0, cnt)
template <typename OffT>
__global__ void k_piece_row_starts(int64_t lo, int64_t cnt_rows, int64_t arcs, int sb, const uint64_t *key,
                                   uint64_t off, OffT *rs) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt_rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t target = (uint64_t)i << sb;
        int64_t a = 0, b = arcs;
        while (a < b) {
            const int64_t mid = (a + b) >> 1;
            if (key[mid] < target) a = mid + 1; else b = mid;
        }
        rs[lo + i] = (OffT)(off + (uint64_t)a);
    }
}

// dedup flags of a piece: keys hold (src - lo) << sb | dst
__global__ void k_piece_dedup_flags(int64_t arcs, int sb, int64_t lo, const uint64_t *key, uint8_t *keep) {
    const uint64_t mask = (uint64_t(1) << sb) - 1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < arcs;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = key[i];
        const bool self = (k >> sb) + (uint64_t)lo == (k & mask);
        const bool dup = i > 0 && key[i - 1] == k;
        keep[i] = !(self || dup);
    }
}

__global__ void k_key_to_adj_off(int64_t arcs, int sb, const uint64_t *key, uint32_t *adj) {
    const uint64_t mask = (uint64_t(1) << sb) - 1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < arcs;
         i += (int64_t)gridDim.x * blockDim.x)
        adj[i] = (uint32_t)(key[i] & mask);
}

template <typename OffT>
static int build_pieces(const uint32_t *du, const uint32_t *dv, int64_t m, int64_t n, int dedup, int P,
                        cudaStream_t st, hbfs_graph *g) {
    const int sb = bits_for(n);
    const int64_t span = (n + P - 1) / P;
    const int sl = bits_for(span);
    if (sl + sb > 64) return set_error(HBFS_ECAPACITY, "vertex ids too wide");
    DevBuf cnt;
    HB_CHECK(cnt.alloc(P * 8 + 16));
    HB_CUDA(cudaMemsetAsync(cnt.p, 0, P * 8, st));
    k_piece_counts<<<grid_for(m), 256, P * 8, st>>>(m, du, dv, span, P, cnt.as<unsigned long long>());
    HB_CUDA(cudaGetLastError());
    std::vector<unsigned long long> hc(P);
    HB_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, P * 8, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    unsigned long long mx = 0, tot = 0;
    for (int r = 0; r < P; ++r) {
        mx = std::max(mx, hc[r]);
        tot += hc[r];
    }
    // keep-dup arcs bound the output; dedup only shrinks it
    g->n = n;
    g->m_edges = m;
    g->arcs = (int64_t)tot;
    g->wide = sizeof(OffT) == 8;
    HB_CHECK(alloc_adj(g));
    HB_CHECK(g->rs.alloc((n + 1) * sizeof(OffT)));
    DevBuf k0, k1, tmp, pos, flags, nsel, tmp2;
    HB_CHECK(k0.alloc(mx * 8 + 8));
    HB_CHECK(k1.alloc(mx * 8 + 8));
    HB_CHECK(pos.alloc(16));
    size_t tb = 0;
    {
        cub::DoubleBuffer<uint64_t> db(k0.as<uint64_t>(), k1.as<uint64_t>());
        HB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int64_t)mx, 0, sl + sb, st));
    }
    HB_CHECK(tmp.alloc(tb + 16));
    size_t tb2 = 0;
    if (dedup) {
        HB_CHECK(flags.alloc(mx + 16));
        HB_CHECK(nsel.alloc(16));
        HB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb2, k0.as<uint64_t>(), flags.as<uint8_t>(),
                                           k1.as<uint64_t>(), nsel.as<int64_t>(), (int64_t)mx, st));
        HB_CHECK(tmp2.alloc(tb2 + 16));
    }
    uint64_t off = 0;
    for (int r = 0; r < P; ++r) {
        const int64_t lo = r * span, rows = std::max<int64_t>(0, std::min<int64_t>(span, n - lo));
        if (rows == 0) continue;
        int64_t c = (int64_t)hc[r];
        HB_CUDA(cudaMemsetAsync(pos.p, 0, 8, st));
        k_piece_keys<<<grid_for(m), 256, 0, st>>>(m, du, dv, lo, span, sb, k0.as<uint64_t>(),
                                                  pos.as<unsigned long long>());
        HB_CUDA(cudaGetLastError());
        cub::DoubleBuffer<uint64_t> db(k0.as<uint64_t>(), k1.as<uint64_t>());
        size_t t = tb;
        if (c > 0) HB_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, t, db, c, 0, sl + sb, st));
        uint64_t *sorted = db.Current();
        if (dedup && c > 0) {
            uint64_t *other = db.Alternate();
            k_piece_dedup_flags<<<grid_for(c), 256, 0, st>>>(c, sb, lo, sorted, flags.as<uint8_t>());
            HB_CUDA(cudaGetLastError());
            size_t t2 = tb2;
            HB_CUDA(cub::DeviceSelect::Flagged(tmp2.p, t2, sorted, flags.as<uint8_t>(), other,
                                               nsel.as<int64_t>(), c, st));
            int64_t h = 0;
            HB_CUDA(cudaMemcpyAsync(&h, nsel.p, 8, cudaMemcpyDeviceToHost, st));
            HB_CUDA(cudaStreamSynchronize(st));
            c = h;
            sorted = other;
        }
        if (c > 0) {
            k_key_to_adj_off<<<grid_for(c), 256, 0, st>>>(c, sb, sorted, g->adj.as<uint32_t>() + off);
            HB_CUDA(cudaGetLastError());
        }
        k_piece_row_starts<OffT><<<grid_for(rows), 256, 0, st>>>(lo, rows, c, sb, sorted, off, g->rs.as<OffT>());
        HB_CUDA(cudaGetLastError());
        off += (uint64_t)c;
        HB_CUDA(cudaStreamSynchronize(st));  // k0/k1 are reused by the next piece
    }
    g->arcs = (int64_t)off;
    if (g->wide) {
        const uint64_t e = off;
        HB_CUDA(cudaMemcpyAsync(g->rs.as<uint64_t>() + n, &e, 8, cudaMemcpyHostToDevice, st));
    } else {
        const uint32_t e = (uint32_t)off;
        HB_CUDA(cudaMemcpyAsync(g->rs.as<uint32_t>() + n, &e, 4, cudaMemcpyHostToDevice, st));
    }
    HB_CUDA(cudaStreamSynchronize(st));
    return graph_finalize(g, st);
}

static int build_from_edges_dev(const uint32_t *du, const uint32_t *dv, int64_t m, int64_t n,
                                int dedup, cudaStream_t st, hbfs_graph *g) {
    const int sb = bits_for(n);
    if (2 * sb > 64) return set_error(HBFS_ECAPACITY, "vertex ids too wide");
    int64_t arcs = 2 * m;
    {
        // monolithic sort: 2 key buffers + adjacency + sort scratch; otherwise
        // the source-range build with as many pieces as the free memory needs
        size_t fr = 0, total = 0;
        cudaMemGetInfo(&fr, &total);
        const int64_t force = getenv("HBFS_BUILD_PIECES") ? atoll(getenv("HBFS_BUILD_PIECES")) : 0;
        const double need = (double)arcs * (8 + 8 + 4 + 1) + (double)(n + 1) * 8;
        if (m > 0 && (force > 1 || need > 0.85 * (double)fr)) {
            int P = force > 1 ? (int)force : 2;
            while (force <= 1 && P < 1024 &&
                   (double)arcs * 4 + (double)arcs / P * (8 + 8 + 1) * 1.3 + (double)(n + 1) * 8 > 0.85 * (double)fr)
                P *= 2;
            const bool wide = arcs >= (int64_t(1) << 32) - 1024;
            return wide ? build_pieces<uint64_t>(du, dv, m, n, dedup, P, st, g)
                        : build_pieces<uint32_t>(du, dv, m, n, dedup, P, st, g);
        }
    }
    DevBuf k0, k1, tmp;
    HB_CHECK(k0.alloc(arcs * 8 + 8));
    HB_CHECK(k1.alloc(arcs * 8 + 8));
    if (m > 0) {
        k_arc_keys<<<grid_for(m), 256, 0, st>>>(m, sb, du, dv, k0.as<uint64_t>());
        HB_CUDA(cudaGetLastError());
        cub::DoubleBuffer<uint64_t> db(k0.as<uint64_t>(), k1.as<uint64_t>());
        size_t tb = 0;
        HB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, arcs, 0, 2 * sb, st));
        HB_CHECK(tmp.alloc(tb));
        HB_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, db, arcs, 0, 2 * sb, st));
        uint64_t *sorted = db.Current();
        uint64_t *other = db.Alternate();
        if (dedup) {
            DevBuf flags, nsel, tmp2;
            HB_CHECK(flags.alloc(arcs));
            HB_CHECK(nsel.alloc(8));
            k_dedup_flags<<<grid_for(arcs), 256, 0, st>>>(arcs, sb, sorted, flags.as<uint8_t>());
            HB_CUDA(cudaGetLastError());
            size_t tb2 = 0;
            HB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb2, sorted, flags.as<uint8_t>(), other,
                                               nsel.as<int64_t>(), arcs, st));
            HB_CHECK(tmp2.alloc(tb2));
            HB_CUDA(cub::DeviceSelect::Flagged(tmp2.p, tb2, sorted, flags.as<uint8_t>(), other,
                                               nsel.as<int64_t>(), arcs, st));
            int64_t h = 0;
            HB_CUDA(cudaMemcpyAsync(&h, nsel.p, 8, cudaMemcpyDeviceToHost, st));
            HB_CUDA(cudaStreamSynchronize(st));
            arcs = h;
            sorted = other;
        }
        g->n = n;
        g->arcs = arcs;
        g->m_edges = m;
        g->wide = arcs >= (int64_t(1) << 32) - 1024;  // 32-bit offsets keep 1024 of headroom
        HB_CHECK(alloc_adj(g));
        k_key_to_adj<<<grid_for(arcs), 256, 0, st>>>(arcs, sb, sorted, g->adj.as<uint32_t>());
        HB_CUDA(cudaGetLastError());
        if (g->wide) {
            HB_CHECK(g->rs.alloc((n + 1) * 8));
            k_row_starts<uint64_t><<<grid_for(n + 1), 256, 0, st>>>(n, arcs, sb, sorted, g->rs.as<uint64_t>());
        } else {
            HB_CHECK(g->rs.alloc((n + 1) * 4));
            k_row_starts<uint32_t><<<grid_for(n + 1), 256, 0, st>>>(n, arcs, sb, sorted, g->rs.as<uint32_t>());
        }
        HB_CUDA(cudaGetLastError());
        HB_CUDA(cudaStreamSynchronize(st));
    } else {
        g->n = n;
        g->arcs = 0;
        g->m_edges = 0;
        g->wide = 0;
        HB_CHECK(alloc_adj(g));
        HB_CHECK(g->rs.alloc((n + 1) * 4));
        HB_CUDA(cudaMemsetAsync(g->rs.p, 0, (n + 1) * 4, st));
    }
    return graph_finalize(g, st);
}

// --------------------------------------------------------- source sampling

__global__ void k_eligible(int64_t n, const uint32_t *order, const void *rs, int wide,
                           uint8_t *flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = order[i];
        uint64_t d;
        if (wide) {
            const uint64_t *r = (const uint64_t *)rs;
            d = r[v + 1] - r[v];
        } else {
            const uint32_t *r = (const uint32_t *)rs;
            d = r[v + 1] - r[v];
        }
        flag[i] = d > 0;
    }
}

}  // namespace hbfs

// =================================================================== C ABI

using namespace hbfs;

extern "C" int hbfs_version(void) { return 100; }

extern "C" const char *hbfs_last_error(void) { return g_err.c_str(); }

extern "C" int hbfs_graph_from_csr(const int64_t *row_starts, const uint32_t *adjacency,
                                   int64_t n, int64_t m_edges, int on_device, void *stream,
                                   hbfs_graph **out) {
    HB_ENTRY_BEGIN
    clear_error();
    if (!out || !row_starts || n < 0) return set_error(HBFS_EINVAL, "bad arguments");
    if (n > (int64_t(1) << 32)) return set_error(HBFS_ECAPACITY, "vertex ids are 32-bit");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int64_t arcs = 0;
    if (on_device)
        HB_CUDA(cudaMemcpy(&arcs, row_starts + n, 8, cudaMemcpyDeviceToHost));
    else
        arcs = row_starts[n];
    if (arcs < 0) return set_error(HBFS_EINVAL, "negative arc count");
    hbfs_graph *g = new hbfs_graph();
    g->n = n;
    g->arcs = arcs;
    g->m_edges = m_edges;
    g->wide = arcs >= (int64_t(1) << 32) - 1024;  // 32-bit offsets keep 1024 of headroom
    int rc = alloc_adj(g);
    DevBuf rs64;
    if (!rc) rc = rs64.alloc((n + 1) * 8);
    if (!rc) rc = g->rs.alloc((n + 1) * (g->wide ? 8 : 4));
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (!rc && cudaMemcpyAsync(rs64.p, row_starts, (n + 1) * 8, kind, st) != cudaSuccess)
        rc = set_error(HBFS_ECUDA, "row_starts copy failed");
    if (!rc && arcs > 0 && cudaMemcpyAsync(g->adj.p, adjacency, arcs * 4, kind, st) != cudaSuccess)
        rc = set_error(HBFS_ECUDA, "adjacency copy failed");
    if (!rc) {
        DevBuf bad;
        unsigned hbad = 0;
        rc = bad.alloc(4);
        if (!rc && (cudaMemsetAsync(bad.p, 0, 4, st) != cudaSuccess))
            rc = set_error(HBFS_ECUDA, "memset failed");
        if (!rc) {
            k_check_csr<<<grid_for(std::max<int64_t>(n, arcs)), 256, 0, st>>>(
                n, arcs, rs64.as<int64_t>(), g->adj.as<uint32_t>(), bad.as<unsigned>());
            if (cudaGetLastError() != cudaSuccess ||
                cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                cudaStreamSynchronize(st) != cudaSuccess)
                rc = set_error(HBFS_ECUDA, "CSR check failed");
        }
        if (!rc && hbad)
            rc = set_error(HBFS_EINVAL, "invalid CSR:%s%s%s", (hbad & 1) ? " row_starts[0] != 0" : "",
                           (hbad & 2) ? " row_starts not non-decreasing" : "",
                           (hbad & 4) ? " adjacency id >= n" : "");
    }
    if (!rc) {
        if (g->wide)
            cudaMemcpyAsync(g->rs.p, rs64.p, (n + 1) * 8, cudaMemcpyDeviceToDevice, st);
        else
            k_narrow<<<grid_for(n + 1), 256, 0, st>>>(n + 1, rs64.as<int64_t>(), g->rs.as<uint32_t>());
        if (cudaGetLastError() != cudaSuccess) rc = set_error(HBFS_ECUDA, "narrow failed");
    }
    if (!rc) rc = graph_finalize(g, st);
    if (rc) {
        delete g;
        return rc;
    }
    *out = g;
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_graph_build(const uint32_t *u, const uint32_t *v, int64_t m, int64_t n,
                                int dedup, int on_device, void *stream, hbfs_graph **out) {
    HB_ENTRY_BEGIN
    clear_error();
    if (!out || m < 0 || n < 0) return set_error(HBFS_EINVAL, "bad arguments");
    if (n > (int64_t(1) << 32)) return set_error(HBFS_ECAPACITY, "vertex ids are 32-bit");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    DevBuf du, dv;
    const uint32_t *pu = u, *pv = v;
    if (!on_device && m > 0) {
        HB_CHECK(du.alloc(m * 4));
        HB_CHECK(dv.alloc(m * 4));
        HB_CUDA(cudaMemcpyAsync(du.p, u, m * 4, cudaMemcpyHostToDevice, st));
        HB_CUDA(cudaMemcpyAsync(dv.p, v, m * 4, cudaMemcpyHostToDevice, st));
        pu = du.as<uint32_t>();
        pv = dv.as<uint32_t>();
    }
    hbfs_graph *g = new hbfs_graph();
    int rc = build_from_edges_dev(pu, pv, m, n, dedup, st, g);
    if (rc) {
        delete g;
        return rc;
    }
    *out = g;
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_generate_edges(int scale, int64_t edgefactor, uint64_t seed,
                                   const double thresholds[3], int permute, uint32_t *u,
                                   uint32_t *v, int on_device, void *stream) {
    HB_ENTRY_BEGIN
    clear_error();
    if (scale < 0 || scale > 32 || edgefactor < 1 || !thresholds)
        return set_error(HBFS_EINVAL, "bad generator parameters");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t m = (int64_t(1) << scale) * edgefactor;
    if (on_device) {
        HB_CHECK(gen_edges_dev(scale, edgefactor, seed, thresholds, permute, u, v, st));
        HB_CUDA(cudaStreamSynchronize(st));
        return HBFS_OK;
    }
    DevBuf du, dv;
    HB_CHECK(du.alloc(m * 4));
    HB_CHECK(dv.alloc(m * 4));
    HB_CHECK(gen_edges_dev(scale, edgefactor, seed, thresholds, permute, du.as<uint32_t>(),
                           dv.as<uint32_t>(), st));
    HB_CUDA(cudaMemcpyAsync(u, du.p, m * 4, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaMemcpyAsync(v, dv.p, m * 4, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_graph_generate(int scale, int64_t edgefactor, uint64_t seed,
                                   const double thresholds[3], int permute, int dedup,
                                   void *stream, hbfs_graph **out) {
    HB_ENTRY_BEGIN
    clear_error();
    if (!out || scale < 0 || scale > 32 || edgefactor < 1 || !thresholds)
        return set_error(HBFS_EINVAL, "bad generator parameters");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t n = int64_t(1) << scale;
    const int64_t m = n * edgefactor;
    DevBuf du, dv;
    HB_CHECK(du.alloc(m * 4));
    HB_CHECK(dv.alloc(m * 4));
    HB_CHECK(gen_edges_dev(scale, edgefactor, seed, thresholds, permute, du.as<uint32_t>(),
                           dv.as<uint32_t>(), st));
    hbfs_graph *g = new hbfs_graph();
    int rc = build_from_edges_dev(du.as<uint32_t>(), dv.as<uint32_t>(), m, n, dedup, st, g);
    if (rc) {
        delete g;
        return rc;
    }
    *out = g;
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_graph_info(const hbfs_graph *g, int64_t *n, int64_t *arcs, int64_t *m_edges,
                               int64_t *max_degree, int32_t *wide_offsets) {
    if (!g) return set_error(HBFS_EINVAL, "null graph");
    if (n) *n = g->n;
    if (arcs) *arcs = g->arcs;
    if (m_edges) *m_edges = g->m_edges;
    if (max_degree) *max_degree = g->max_degree;
    if (wide_offsets) *wide_offsets = g->wide;
    return HBFS_OK;
}

extern "C" int hbfs_graph_export(const hbfs_graph *g, int64_t *row_starts, uint32_t *adjacency,
                                 int on_device, void *stream) {
    HB_ENTRY_BEGIN
    clear_error();
    if (!g) return set_error(HBFS_EINVAL, "null graph");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t n = g->n;
    if (row_starts) {
        DevBuf tmp;
        int64_t *dst = row_starts;
        if (!on_device) {
            HB_CHECK(tmp.alloc((n + 1) * 8));
            dst = tmp.as<int64_t>();
        }
        if (g->wide)
            k_widen<uint64_t><<<grid_for(n + 1), 256, 0, st>>>(n + 1, g->rs.as<uint64_t>(), dst);
        else
            k_widen<uint32_t><<<grid_for(n + 1), 256, 0, st>>>(n + 1, g->rs.as<uint32_t>(), dst);
        HB_CUDA(cudaGetLastError());
        if (!on_device)
            HB_CUDA(cudaMemcpyAsync(row_starts, dst, (n + 1) * 8, cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaStreamSynchronize(st));
    }
    if (adjacency && g->arcs > 0) {
        HB_CUDA(cudaMemcpyAsync(adjacency, g->adj.p, g->arcs * 4,
                                on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaStreamSynchronize(st));
    }
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_graph_free(hbfs_graph *g) {
    HB_ENTRY_BEGIN
    delete g;
    return HBFS_OK;
    HB_ENTRY_END
}

// ids whose source-order key lies below `limit`, appended in any order
__global__ void k_order_below(int64_t n, uint64_t seed, uint64_t limit, unsigned long long *cnt, int64_t cap,
                              uint32_t *ids, uint64_t *keys) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = hbfs::mix64(hbfs::mix64((uint64_t)i + 0x5EEDu) ^ seed);
        if (k < limit) {
            const unsigned long long at = atomicAdd(cnt, 1ull);
            if ((int64_t)at < cap) {
                ids[at] = (uint32_t)i;
                keys[at] = k;
            }
        }
    }
}

// The first `count` ids of the source sampling order argsort(mix64(mix64(id +
// 0x5EED) ^ seed)) (harness.py:85-87) without sorting all n keys or touching
// a graph: the keys are uniform, so a threshold keeps about 4 * count of them.
// For partitioned graphs (mgpu.sample_sources_partitioned), where no rank
// holds every degree.
extern "C" int hbfs_source_order_prefix(int64_t n, uint64_t seed, int64_t count, uint32_t *out) {
    HB_ENTRY_BEGIN
    clear_error();
    if (!out || count < 0 || count > n) return set_error(HBFS_EINVAL, "bad arguments");
    if (count == 0) return HBFS_OK;
    const int64_t cap = 8 * count + 1024;
    DevBuf cnt, ids, keys;
    HB_CHECK(cnt.alloc(8));
    HB_CHECK(ids.alloc(cap * 4));
    HB_CHECK(keys.alloc(cap * 8));
    std::vector<uint32_t> hi(cap);
    std::vector<uint64_t> hk(cap);
    for (double want = 4.0 * (double)count + 256;; want *= 2) {
        const double frac = want / (double)n;
        const uint64_t limit = frac >= 1.0 ? ~0ull : (uint64_t)(frac * 18446744073709551615.0);
        HB_CUDA(cudaMemset(cnt.p, 0, 8));
        k_order_below<<<grid_for(n), 256>>>(n, seed, limit, cnt.as<unsigned long long>(), cap, ids.as<uint32_t>(),
                                          keys.as<uint64_t>());
        HB_CUDA(cudaGetLastError());
        unsigned long long got = 0;
        HB_CUDA(cudaMemcpy(&got, cnt.p, 8, cudaMemcpyDeviceToHost));
        if ((int64_t)got > cap) return set_error(HBFS_ECUDA, "source order: threshold kept too many keys");
        if ((int64_t)got < count && limit != ~0ull) continue;  // too few: widen
        HB_CUDA(cudaMemcpy(hi.data(), ids.p, got * 4, cudaMemcpyDeviceToHost));
        HB_CUDA(cudaMemcpy(hk.data(), keys.p, got * 8, cudaMemcpyDeviceToHost));
        std::vector<int64_t> idx(got);
        for (size_t i = 0; i < got; ++i) idx[i] = (int64_t)i;
        std::sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
            return hk[a] != hk[b] ? hk[a] < hk[b] : hi[a] < hi[b];
        });
        for (int64_t i = 0; i < count; ++i) out[i] = hi[idx[i]];
        return HBFS_OK;
    }
    HB_ENTRY_END
}

extern "C" int hbfs_sample_sources(const hbfs_graph *g, int64_t count, uint64_t seed,
                                   int allow_isolated, uint32_t *out) {
    HB_ENTRY_BEGIN
    clear_error();
    if (!g || !out || count < 0) return set_error(HBFS_EINVAL, "bad arguments");
    const int64_t n = g->n;
    if (count > n)
        return set_error(HBFS_EINVAL, "cannot sample %lld distinct vertices from %lld",
                         (long long)count, (long long)n);
    if (count == 0) return HBFS_OK;
    cudaStream_t st = 0;
    DevBuf order;
    HB_CHECK(order.alloc(n * 4));
    HB_CHECK(keyed_order(n, seed, 0x5EED, order.as<uint32_t>(), st));
    if (allow_isolated) {
        HB_CUDA(cudaMemcpy(out, order.p, count * 4, cudaMemcpyDeviceToHost));
        return HBFS_OK;
    }
    DevBuf flags, sel, nsel, tmp;
    HB_CHECK(flags.alloc(n));
    HB_CHECK(sel.alloc(n * 4));
    HB_CHECK(nsel.alloc(8));
    k_eligible<<<grid_for(n), 256, 0, st>>>(n, order.as<uint32_t>(), g->rs.p, g->wide,
                                            flags.as<uint8_t>());
    HB_CUDA(cudaGetLastError());
    size_t tb = 0;
    HB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, order.as<uint32_t>(), flags.as<uint8_t>(),
                                       sel.as<uint32_t>(), nsel.as<int64_t>(), n, st));
    HB_CHECK(tmp.alloc(tb));
    HB_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, order.as<uint32_t>(), flags.as<uint8_t>(),
                                       sel.as<uint32_t>(), nsel.as<int64_t>(), n, st));
    int64_t k = 0;
    HB_CUDA(cudaMemcpy(&k, nsel.p, 8, cudaMemcpyDeviceToHost));
    if (k < count)
        return set_error(HBFS_EINVAL, "only %lld vertices with degree >= 1, need %lld",
                         (long long)k, (long long)count);
    HB_CUDA(cudaMemcpy(out, sel.p, count * 4, cudaMemcpyDeviceToHost));
    return HBFS_OK;
    HB_ENTRY_END
}
