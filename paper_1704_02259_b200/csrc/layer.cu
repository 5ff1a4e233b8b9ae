// Per-layer kernels and the sequential-order reference BFS, on device buffers.
//
// The reference's compiled module hybfs._native exposes its layer steps to the
// engine glue and to its tests: top_down_layer,
// top_down_chunked, bottom_up_layer, bottom_up_multiple_set and bfs_reference
// (_native.pyx:39-239).  These entry points keep their in-place contract on
// caller-owned bitmaps (vis, out) and parent arrays, with int64 row starts as
// in the reference, so the reference's per-layer tests can run against the
// GPU.  The production traversal is the persistent kernel of bfs.cu; these are
// plain grid kernels — correct first, then reasonably parallel.
//
// Results are the reference's, bit for bit:
//  * top-down: the sequential loop claims v for the first frontier u in
//    ascending order (_native.pyx:65-86), i.e. parent = min frontier u over
//    arcs into v unvisited at layer start -> atomicMin into a candidate array;
//  * bottom-up: v takes the first frontier entry of its sorted row
//    (_native.pyx:89-104); the 16-lane variant gives the same parents plus its
//    gather/fallback counters (_native.pyx:107-204);
//  * bfs_reference: parent = the first discoverer in FIFO-queue order
//    (_native.pyx:39-62).  The queue order of level d+1 is the lexicographic
//    order of (queue position of the first discoverer, row position), so each
//    level is one atomicMin over 64-bit keys plus a radix sort of the level.
#include <cub/cub.cuh>

#include "common.cuh"

namespace hbfs {
namespace {

constexpr int kLB = 256;
constexpr uint32_t kCandNone = 0xFFFFFFFFu;

inline int lgrid(int64_t items) {
    int64_t g = (items + kLB - 1) / kLB;
    if (g > 148 * 16) g = 148 * 16;
    return (int)(g < 1 ? 1 : g);
}

#define LSTRIDE(i, N) \
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (N); i += (int64_t)gridDim.x * blockDim.x)

__device__ __forceinline__ bool tbit(const uint32_t *w, uint64_t v) { return (w[v >> 5] >> (v & 31)) & 1u; }

// Frontier queue from a bitmap (ascending within a word; order is irrelevant
// to the results) plus the frontier degree sum (top_down_chunked's gathers).
__global__ void kl_queue(int64_t nw, int64_t n, const uint32_t *inw, const int64_t *rs, uint32_t *q,
                         unsigned long long *cnt) {
    LSTRIDE(w, nw) {
        uint32_t bits = inw[w];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int64_t u = w * 32 + b;
            if (u >= n) break;
            q[atomicAdd(&cnt[0], 1ull)] = (uint32_t)u;
            atomicAdd(&cnt[1], (unsigned long long)(rs[u + 1] - rs[u]));
        }
    }
}

// Top-down expansion: warp per frontier vertex; every arc into a vertex not
// visited at layer start lowers cand[v] and marks v in `nb` (new bits).
__global__ void kl_td(const uint32_t *q, int64_t qn, const int64_t *rs, const uint32_t *adj,
                      const uint32_t *vis, uint32_t *cand, uint32_t *nb) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < qn;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t u = q[i];
        for (int64_t k = rs[u] + lane; k < rs[u + 1]; k += 32) {
            const uint32_t v = adj[k];
            if (tbit(vis, v)) continue;
            atomicMin(&cand[v], u);
            const uint32_t b = 1u << (v & 31);
            if (!(__ldcg(&nb[v >> 5]) & b)) atomicOr(&nb[v >> 5], b);
        }
    }
}

// Commit the claims: vis |= nb, out |= nb, parent = cand; reset the scratch.
__global__ void kl_td_commit(int64_t nw, uint32_t *nb, uint32_t *cand, uint32_t *vis, uint32_t *out,
                             uint32_t *parent) {
    LSTRIDE(w, nw) {
        const uint32_t bits = nb[w];
        if (!bits) continue;
        nb[w] = 0;
        vis[w] |= bits;
        out[w] |= bits;
        for (uint32_t x = bits; x; x &= x - 1) {
            const int64_t v = w * 32 + __ffs(x) - 1;
            parent[v] = cand[v];
            cand[v] = kCandNone;
        }
    }
}

// Bottom-up: lane per vertex of a word; the first frontier entry of the row
// wins (warp-cooperative scan for rows left open after max_pos entries).
// Counters follow the 16-lane kernel: gathers = pos+1 for a hit at pos <
// max_pos, else min(deg, max_pos); fallback when deg > max_pos and no hit
// among the first max_pos entries.
__global__ void kl_bu(int64_t nw, int64_t n, const int64_t *rs, const uint32_t *adj, const uint32_t *inw,
                      uint32_t *vis, uint32_t *out, uint32_t *parent, int64_t max_pos,
                      unsigned long long *ctr) {
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    unsigned long long c_gat = 0, c_fb = 0;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t vw = vis[w];
        const int64_t v = w * 32 + lane;
        const bool valid = v < n;
        const int64_t s = valid ? rs[v] : 0, e = valid ? rs[v + 1] : 0;
        const bool mine = valid && !((vw >> lane) & 1u) && e > s;
        int64_t hit = -1, p = s;
        uint32_t hu = 0;
        if (mine) {
            for (int it = 0; it < 8 && p < e; ++it, ++p) {
                const uint32_t a = adj[p];
                if (tbit(inw, a)) {
                    hit = p;
                    hu = a;
                    break;
                }
            }
        }
        unsigned todo = __ballot_sync(full, mine && hit < 0 && p < e);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const int64_t ps = __shfl_sync(full, (long long)p, src), pe = __shfl_sync(full, (long long)e, src);
            int64_t h = -1;
            uint32_t hv = 0;
            for (int64_t c = ps; c < pe; c += 32) {
                const int64_t k = c + lane;
                const uint32_t a = k < pe ? adj[k] : 0u;
                const unsigned bb = __ballot_sync(full, k < pe && tbit(inw, a));
                if (bb) {
                    const int l = __ffs(bb) - 1;
                    h = c + l;
                    hv = __shfl_sync(full, a, l);
                    break;
                }
            }
            if (lane == src) {
                hit = h;
                hu = hv;
            }
        }
        const bool found = hit >= 0;
        if (found) parent[v] = hu;
        const unsigned fm = __ballot_sync(full, found);
        if (lane == 0 && fm) {
            vis[w] = vw | fm;
            out[w] |= fm;
        }
        if (mine) {
            const int64_t deg = e - s, pos = found ? hit - s : -1;
            const bool early = found && pos < max_pos;
            c_gat += (unsigned long long)(early ? pos + 1 : (deg < max_pos ? deg : max_pos));
            c_fb += (deg > max_pos && !early) ? 1ull : 0ull;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        c_gat += __shfl_down_sync(full, c_gat, o);
        c_fb += __shfl_down_sync(full, c_fb, o);
    }
    if (lane == 0) {
        if (c_fb) atomicAdd(&ctr[0], c_fb);
        if (c_gat) atomicAdd(&ctr[1], c_gat);
    }
}

__global__ void kl_fill_u32(uint32_t *p, int64_t n, uint32_t x) {
    LSTRIDE(i, n) p[i] = x;
}
__global__ void kl_fill_u64(unsigned long long *p, int64_t n, unsigned long long x) {
    LSTRIDE(i, n) p[i] = x;
}

// ---- reference BFS (FIFO order) ----

__global__ void kl_ref_init(int64_t n, uint32_t source, uint32_t *parent, int32_t *level, uint32_t *queue) {
    LSTRIDE(i, n) {
        parent[i] = i == (int64_t)source ? source : HBFS_NIL;
        level[i] = i == (int64_t)source ? 0 : -1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) queue[0] = source;
}

// Level expansion in queue order: key(v) = min over arcs (queue position of
// u) << 32 | (row position); the first arc into v lists it for the sort.
__global__ void kl_ref_expand(const uint32_t *queue, int64_t head, int64_t tail, const int64_t *rs,
                              const uint32_t *adj, const int32_t *level, unsigned long long *key,
                              uint32_t *listed, uint32_t *next, unsigned long long *cnt) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = head + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < tail;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t u = queue[i];
        const int64_t s = rs[u], e = rs[u + 1];
        for (int64_t k = s + lane; k < e; k += 32) {
            const uint32_t v = adj[k];
            if (level[v] != -1) continue;
            atomicMin(&key[v], ((unsigned long long)i << 32) | (unsigned long long)(k - s));
            const uint32_t b = 1u << (v & 31);
            if (__ldcg(&listed[v >> 5]) & b) continue;
            if (atomicOr(&listed[v >> 5], b) & b) continue;
            next[atomicAdd(cnt, 1ull)] = v;
        }
    }
}

__global__ void kl_ref_keys(const uint32_t *next, int64_t c, const unsigned long long *key,
                            unsigned long long *k_out) {
    LSTRIDE(i, c) k_out[i] = key[next[i]];
}

// Sorted level -> queue slots, parents (queue[key >> 32]), levels; reset scratch.
__global__ void kl_ref_commit(const uint32_t *vs, const unsigned long long *ks, int64_t c, int64_t tail,
                              int32_t depth1, uint32_t *queue, uint32_t *parent, int32_t *level,
                              unsigned long long *key, uint32_t *listed) {
    LSTRIDE(i, c) {
        const uint32_t v = vs[i];
        queue[tail + i] = v;
        parent[v] = queue[ks[i] >> 32];
        level[v] = depth1;
        key[v] = ~0ull;
        listed[v >> 5] = 0u;
    }
}

// Scratch owned by the calling thread: grown on demand, reused across calls.
struct LayerScratch {
    int64_t n = -1;
    DevBuf cand, nb, q, cnt;
    int ensure(int64_t n_) {
        if (n_ <= n) return HBFS_OK;
        const int64_t nw = (n_ + 31) / 32;
        HB_CHECK(cand.alloc(n_ * 4 + 16));
        HB_CHECK(nb.alloc(nw * 4 + 16));
        HB_CHECK(q.alloc(n_ * 4 + 16));
        HB_CHECK(cnt.alloc(64));
        kl_fill_u32<<<lgrid(n_), kLB>>>(cand.as<uint32_t>(), n_, kCandNone);
        HB_CUDA(cudaMemset(nb.p, 0, nw * 4 + 16));
        HB_CUDA(cudaDeviceSynchronize());
        n = n_;
        return HBFS_OK;
    }
};
thread_local LayerScratch t_scratch;

int check_layer_args(const int64_t *rs, const uint32_t *adj, const uint32_t *inw, uint32_t *vis,
                     uint32_t *out, uint32_t *parent, int64_t n) {
    if (n < 0) return set_error(HBFS_EINVAL, "n must be >= 0");
    if (n > 0 && (!rs || !inw || !vis || !out || !parent))
        return set_error(HBFS_EINVAL, "null buffer");
    if (n >= (int64_t(1) << 32)) return set_error(HBFS_ECAPACITY, "vertex ids are 32-bit");
    (void)adj;
    return HBFS_OK;
}

}  // namespace
}  // namespace hbfs

using namespace hbfs;

extern "C" int hbfs_layer_top_down(const int64_t *rs, const uint32_t *adj, const uint32_t *inw,
                                   uint32_t *vis, uint32_t *out, uint32_t *parent, int64_t n,
                                   int64_t *gathers, void *stream) {
    HB_ENTRY_BEGIN
    clear_error();
    HB_CHECK(check_layer_args(rs, adj, inw, vis, out, parent, n));
    if (gathers) *gathers = 0;
    if (n == 0) return HBFS_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    LayerScratch &S = t_scratch;
    HB_CHECK(S.ensure(n));
    const int64_t nw = (n + 31) / 32;
    unsigned long long *cnt = S.cnt.as<unsigned long long>();
    HB_CUDA(cudaMemsetAsync(cnt, 0, 16, st));
    kl_queue<<<lgrid(nw), kLB, 0, st>>>(nw, n, inw, rs, S.q.as<uint32_t>(), cnt);
    unsigned long long h[2] = {0, 0};
    HB_CUDA(cudaMemcpyAsync(h, cnt, 16, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    if (gathers) *gathers = (int64_t)h[1];
    if (h[0] == 0 || h[1] == 0) return HBFS_OK;
    kl_td<<<lgrid((int64_t)h[0] * 32), kLB, 0, st>>>(S.q.as<uint32_t>(), (int64_t)h[0], rs, adj, vis,
                                                     S.cand.as<uint32_t>(), S.nb.as<uint32_t>());
    kl_td_commit<<<lgrid(nw), kLB, 0, st>>>(nw, S.nb.as<uint32_t>(), S.cand.as<uint32_t>(), vis, out, parent);
    HB_CUDA(cudaGetLastError());
    HB_CUDA(cudaStreamSynchronize(st));
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_layer_bottom_up(const int64_t *rs, const uint32_t *adj, const uint32_t *inw,
                                    uint32_t *vis, uint32_t *out, uint32_t *parent, int64_t n,
                                    int32_t max_pos, int64_t *fallback, int64_t *gathers,
                                    void *stream) {
    HB_ENTRY_BEGIN
    clear_error();
    HB_CHECK(check_layer_args(rs, adj, inw, vis, out, parent, n));
    if (max_pos < 1) return set_error(HBFS_EINVAL, "max_pos must be >= 1");
    if (fallback) *fallback = 0;
    if (gathers) *gathers = 0;
    if (n == 0) return HBFS_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    LayerScratch &S = t_scratch;
    HB_CHECK(S.ensure(n));
    const int64_t nw = (n + 31) / 32;
    unsigned long long *cnt = S.cnt.as<unsigned long long>();
    HB_CUDA(cudaMemsetAsync(cnt, 0, 16, st));
    kl_bu<<<lgrid(nw * 32), kLB, 0, st>>>(nw, n, rs, adj, inw, vis, out, parent, max_pos, cnt);
    HB_CUDA(cudaGetLastError());
    unsigned long long h[2] = {0, 0};
    HB_CUDA(cudaMemcpyAsync(h, cnt, 16, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    if (fallback) *fallback = (int64_t)h[0];
    if (gathers) *gathers = (int64_t)h[1];
    return HBFS_OK;
    HB_ENTRY_END
}

extern "C" int hbfs_reference_bfs(const int64_t *rs, const uint32_t *adj, int64_t n, int64_t source,
                                  uint32_t *parent, int32_t *level, void *stream) {
    HB_ENTRY_BEGIN
    clear_error();
    if (n <= 0 || !rs || !parent || !level) return set_error(HBFS_EINVAL, "bad arguments");
    if (source < 0 || source >= n)
        return set_error(HBFS_ERANGE, "source %lld out of range [0, %lld)", (long long)source, (long long)n);
    if (n >= (int64_t(1) << 32)) return set_error(HBFS_ECAPACITY, "vertex ids are 32-bit");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t nw = (n + 31) / 32;
    DevBuf queue, key, listed, next, ks, ks2, vs2, cnt, tmp;
    HB_CHECK(queue.alloc(n * 4 + 16));
    HB_CHECK(key.alloc(n * 8 + 16));
    HB_CHECK(listed.alloc(nw * 4 + 16));
    HB_CHECK(next.alloc(n * 4 + 16));
    HB_CHECK(ks.alloc(n * 8 + 16));
    HB_CHECK(ks2.alloc(n * 8 + 16));
    HB_CHECK(vs2.alloc(n * 4 + 16));
    HB_CHECK(cnt.alloc(16));
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (const unsigned long long *)nullptr,
                                    (unsigned long long *)nullptr, (const uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (int)std::min<int64_t>(n, INT32_MAX));
    HB_CHECK(tmp.alloc(tmp_bytes + 16));
    kl_fill_u64<<<lgrid(n), kLB, 0, st>>>(key.as<unsigned long long>(), n, ~0ull);
    HB_CUDA(cudaMemsetAsync(listed.p, 0, nw * 4 + 16, st));
    kl_ref_init<<<lgrid(n), kLB, 0, st>>>(n, (uint32_t)source, parent, level, queue.as<uint32_t>());
    HB_CUDA(cudaGetLastError());
    int64_t head = 0, tail = 1;
    for (int32_t d = 0; head < tail; ++d) {
        HB_CUDA(cudaMemsetAsync(cnt.p, 0, 8, st));
        kl_ref_expand<<<lgrid((tail - head) * 32), kLB, 0, st>>>(
            queue.as<uint32_t>(), head, tail, rs, adj, level, key.as<unsigned long long>(),
            listed.as<uint32_t>(), next.as<uint32_t>(), cnt.as<unsigned long long>());
        unsigned long long c = 0;
        HB_CUDA(cudaMemcpyAsync(&c, cnt.p, 8, cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaStreamSynchronize(st));
        if (c == 0) break;
        kl_ref_keys<<<lgrid((int64_t)c), kLB, 0, st>>>(next.as<uint32_t>(), (int64_t)c,
                                                       key.as<unsigned long long>(), ks.as<unsigned long long>());
        size_t tb = tmp_bytes;
        HB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, ks.as<unsigned long long>(),
                                                ks2.as<unsigned long long>(), next.as<uint32_t>(),
                                                vs2.as<uint32_t>(), (int)c, 0, 64, st));
        kl_ref_commit<<<lgrid((int64_t)c), kLB, 0, st>>>(vs2.as<uint32_t>(), ks2.as<unsigned long long>(),
                                                         (int64_t)c, tail, d + 1, queue.as<uint32_t>(),
                                                         parent, level, key.as<unsigned long long>(),
                                                         listed.as<uint32_t>());
        HB_CUDA(cudaGetLastError());
        head = tail;
        tail += (int64_t)c;
    }
    HB_CUDA(cudaStreamSynchronize(st));
    return HBFS_OK;
    HB_ENTRY_END
}
