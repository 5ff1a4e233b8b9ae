// Shared internals of libhbfs.so: error plumbing, the graph object, small
// device helpers.  Nothing here is part of the C ABI (see include/hbfs.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <string>

#include "../../include/hbfs.h"

namespace hbfs {

int set_error(int code, const char *fmt, ...);
void clear_error();

#define HB_CUDA(expr)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return ::hbfs::set_error(HBFS_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr, \
                                     cudaGetErrorString(e_));                           \
    } while (0)

// Device-side index checks (builds with -DHBFS_CHECKED, the bounds-checked
// variant tools/sanitize.py runs): a failed check sets bit `bit` of a device
// flag word (read by hbfs_debug_checks) instead of trapping.
#ifdef HBFS_CHECKED
static __device__ unsigned int g_check_fail = 0;  // per translation unit (no rdc)
#define HB_DCHECK(cond, bit)                                              \
    do {                                                                  \
        if (!(cond)) atomicOr(&::hbfs::g_check_fail, 1u << (bit));        \
    } while (0)
#else
#define HB_DCHECK(cond, bit) \
    do {                     \
    } while (0)
#endif

#define HB_CHECK(expr)                    \
    do {                                  \
        int rc_ = (expr);                 \
        if (rc_ != HBFS_OK) return rc_;   \
    } while (0)

// Guard every C entry point: no C++ exception may cross the ABI.
#define HB_ENTRY_BEGIN try {
#define HB_ENTRY_END                                                           \
    }                                                                          \
    catch (const std::exception &ex) {                                         \
        return ::hbfs::set_error(HBFS_ECUDA, "internal error: %s", ex.what()); \
    }                                                                          \
    catch (...) {                                                              \
        return ::hbfs::set_error(HBFS_ECUDA, "internal error");                \
    }

#ifndef HBFS_KBLOCK
#define HBFS_KBLOCK 512
#endif
constexpr int kBlock = HBFS_KBLOCK;  // threads per CTA for the traversal kernels

struct Workspace;

// Out-of-bounds write detection (compute-sanitizer is not available on the
// GPU pool): with HBFS_GUARD=1 in the environment every DevBuf gets a guard
// band of kGuardBytes filled with kGuardByte behind its end; hbfs_debug_guards
// verifies every live band (a kernel that wrote past an array's end clobbers
// it).  Off by default; no cost when off.
constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kGuardByte = 0xA5;
bool guard_enabled();
void guard_register(void *p, size_t bytes);
void guard_unregister(void *p);

// Device block allocation helper (owned, freed in destructor).
struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    int alloc(size_t b) {
        release();
        if (b == 0) b = 16;
        const bool guard = guard_enabled();
        cudaError_t e = cudaMalloc(&p, b + (guard ? kGuardBytes : 0));
        if (e != cudaSuccess) {
            p = nullptr;
            return set_error(HBFS_ECAPACITY, "cudaMalloc(%zu) failed: %s", b, cudaGetErrorString(e));
        }
        bytes = b;
        if (guard) {
            cudaMemset(static_cast<char *>(p) + b, kGuardByte, kGuardBytes);
            guard_register(p, b);
        }
        return HBFS_OK;
    }
    void release() {
        if (p) {
            guard_unregister(p);
            cudaFree(p);
        }
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T *as() const { return static_cast<T *>(p); }
};

struct Heur {
    int heuristic, counter_mode, force;
    int64_t alpha, beta, n;
};

// Direction rule: hybrid.py:62-80 (reference rule) or Beamer/GAP.  Host+device
// so the controller is identical wherever it runs (persistent kernel, the
// multi-GPU host loop).
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

// Head record of a vertex: its degree and the first kHeadLen entries of its
// sorted row (absent entries = HBFS_NIL), 16 bytes.  The bottom-up layers
// resolve most candidates from this record alone — first hit among the head
// entries, or a row that ends inside the head — without touching the row
// starts or the adjacency array; only rows still open continue at position
// kHeadLen of the CSR row.  The records are packed in rank order over the
// vertices with degree > 0 (`pre[w]` = records before bitmap word w), so the
// candidates of a dense layer read them as contiguous runs.  Built once per
// graph (graph_finalize / part build); synchronises the stream.
constexpr int kHeadLen = 3;
// Second-tier record (32 bytes = one sector, same slot as the head record, stored
// behind the head records in the same buffer at head2_offset): the row start
// and the next row entries — positions kHeadLen .. kHeadLen + 6 with 32-bit
// row offsets (word 0 = row start), kHeadLen .. kHeadLen + 5 with 64-bit ones
// (words 0-1).  A candidate its head record left open continues here: one
// sector instead of the row-start sector plus the row's first adjacency
// sectors, and no dependent row-start load in front of the row.
#ifndef HBFS_H2W
#define HBFS_H2W 8
#endif
constexpr int kH2W = HBFS_H2W;  // words per second-tier record (8 = one sector; 16: experiment)
__host__ __device__ inline int64_t head2_offset(int64_t n_records) {  // in uint4 units, record-aligned
    return (n_records + 4) & ~int64_t(3);
}
int build_heads(int64_t n, const void *rs, int wide, const uint32_t *adj, const uint32_t *posw,
                DevBuf &pre, DevBuf &hd, cudaStream_t st, int64_t *n_records = nullptr);

// A top-down layer whose frontier is only a bitmap (kind 1) runs as a
// bottom-up sweep when at most ratio * e_f candidates are left (unvisited
// vertices with degree > 0): same vertices, same parents (bfs.cu).  Host +
// device: the multi-GPU loop mirrors the kernel's choice.
__host__ __device__ inline bool bu_executes(int dir, int kind, int64_t eu_v, int64_t e_f, int64_t n,
                                            int64_t n_pos, int64_t ratio) {
    const int64_t cand = eu_v - (n - n_pos);
    // few candidates in absolute terms too: a sweep over many candidates behind a
    // small hub frontier scans their rows to the end
    return dir == HBFS_TOP_DOWN && kind == 1 && ratio > 0 && cand <= ratio * e_f && cand * 64 <= n;
}
int64_t bu_exec_ratio();  // HBFS_BU_EXEC_RATIO or the default

// Bottom-up layer of one partition rank with the persistent kernel's tile
// machinery (defined in bfs.cu, used by part.cu).  v_f: global frontier size
// (< 0: unknown).  scratch: part_bu_scratch_bytes() of device memory.
size_t part_bu_scratch_bytes();
int part_bu_launch(const uint64_t *rs_local, const uint32_t *adj, const uint32_t *posw_local,
                   const uint4 *hd_local, int64_t n_pos_local, const uint32_t *pre_local, int64_t n,
                   int64_t lo, int64_t nloc, int64_t arcs_local, const uint32_t *F, uint32_t *V, uint32_t *parent_local,
                   int32_t *level_local, uint32_t *next_slice, int32_t depth, int32_t max_pos, int64_t v_f,
                   unsigned long long *counters, void *scratch, cudaStream_t st);

// Partition traversal with the persistent kernel, one layer per launch
// (bfs.cu; driven by the multi-GPU loop in part.cu).
void *part_trav_create(int64_t n, int64_t lo, int64_t nown, int64_t arcs_local, const uint64_t *rs_local,
                       const uint32_t *adj, const uint32_t *posw_local, const uint4 *hd_local,
                       int64_t n_pos_local, const uint32_t *pre_local, uint32_t *parent_local,
                       int32_t *level_local, uint32_t *cand, uint32_t *touch, int *rc_out, int64_t nw_pad);
void part_trav_free(void *h);
uint32_t *part_trav_plane(void *h, int64_t depth);  // depth < 0: the visited bitmap
int part_trav_levels(void *h, int64_t n_layers, cudaStream_t st);  // final level stamp of the owned vertices
int part_trav_layer(void *h, const int64_t state[6], int32_t dir, int do_init, uint32_t root,
                    const hbfs_params *p, int64_t n_pos_global, unsigned long long *lay_out, int single,
                    cudaStream_t st);  // asynchronous; lay_out (device, may be null): the rank's layer totals
// tot[0..3] += this rank's counters of `layer` (+ applied[0..1], the records it applied), on the stream
int part_trav_add_counters(void *h, int64_t layer, const unsigned long long *applied, unsigned long long *tot,
                           cudaStream_t st);

}  // namespace hbfs

struct hbfs_graph {
    int64_t n = 0;
    int64_t nw = 0;        // bitmap words ceil(n/32)
    int64_t arcs = 0;
    int64_t m_edges = 0;   // TEPS denominator (csr.py:73)
    int64_t max_degree = 0;
    int64_t n_pos = 0;     // vertices with degree > 0 (= head records)
    int wide = 0;          // 1: 64-bit offsets (arcs >= 2^32), else 32-bit
    int device = 0;
    hbfs::DevBuf rs;       // OffT[n+1]
    hbfs::DevBuf adj;      // uint32[arcs + 8] (padded for aligned uint4 reads)
    hbfs::DevBuf posw;     // uint32[nw]: bit v = deg(v) > 0 (engine.py:29-57 `posw`)
    hbfs::DevBuf hd;       // uint4[#deg>0] head records: {deg, row[0], row[1], row[2]} (absent = NIL)
    hbfs::DevBuf pre;      // uint32[nw+1]: head records before bitmap word w
    hbfs::Workspace *ws = nullptr;
    // hbfs_bfs holds this for the whole call: the per-graph workspace (parent,
    // level, bitmaps, queues, controller state, pinned trace mirror) serves one
    // traversal at a time; concurrent callers on one graph serialise here.
    std::mutex mu;
    ~hbfs_graph();
};

namespace hbfs {

// Narrow/widen row starts and derive per-graph metadata (posw, max degree).
int graph_finalize(hbfs_graph *g, cudaStream_t st);

__host__ __device__ inline uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

}  // namespace hbfs
