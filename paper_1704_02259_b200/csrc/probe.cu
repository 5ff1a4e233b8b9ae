// Measurement only: the random-sector read ceiling of this GPU's HBM.
//
// The traversal's DRAM traffic is dominated by 32-byte sectors at data-
// dependent addresses (first sectors of adjacency rows, parent entries), not
// by streams; the copy bandwidth in MEASURED_PEAKS.json is not attainable for
// that pattern.  This kernel measures it the way a bottom-up warp touches
// memory: every warp-iteration picks a random region of 2^log_region bytes of
// a large buffer and its 32 lanes each read one random 32-byte sector inside
// it (two 16-byte loads, evict-first so L2 does not serve repeats).  bench.py
// reports the result next to the copy-bandwidth roofline.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace hbfs {
namespace {

__device__ __forceinline__ uint64_t hsh(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

__global__ void kprobe_sectors(const uint4 *buf, int log_bytes, int log_region, int64_t iters,
                               uint32_t *sink) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t acc = 0;
    for (int64_t i = w; i < iters; i += nw * 4) {
        uint4 v[4][2];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t h = hsh((uint64_t)(i + j * nw));
            const uint64_t region = (h >> 20) & ((1ull << (log_bytes - log_region)) - 1);
            const uint64_t sec = (region << (log_region - 5)) + (hsh(h + lane) & ((1ull << (log_region - 5)) - 1));
            v[j][0] = __ldcs(buf + sec * 2);
            v[j][1] = __ldcs(buf + sec * 2 + 1);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) acc ^= v[j][0].x ^ v[j][1].w;
    }
    if (acc == 0x9E3779B9u) sink[0] = acc;
}

}  // namespace
}  // namespace hbfs

extern "C" int hbfs_probe_random_sectors(int log_bytes, int log_region, double *gbs) {
    HB_ENTRY_BEGIN
    using namespace hbfs;
    clear_error();
    if (!gbs || log_bytes < 20 || log_bytes > 36 || log_region < 6 || log_region > log_bytes)
        return set_error(HBFS_EINVAL, "bad arguments");
    DevBuf buf, sink;
    HB_CHECK(buf.alloc(size_t(1) << log_bytes));
    HB_CHECK(sink.alloc(16));
    HB_CUDA(cudaMemset(buf.p, 1, size_t(1) << log_bytes));
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t iters = int64_t(1) << 22;  // warp-iterations of 32 sectors: 4 GiB
    cudaEvent_t e0, e1;
    HB_CUDA(cudaEventCreate(&e0));
    HB_CUDA(cudaEventCreate(&e1));
    float ms = 0.f;
    for (int rep = 0; rep < 2; ++rep) {
        HB_CUDA(cudaEventRecord(e0));
        kprobe_sectors<<<sms * 8, 256>>>(buf.as<uint4>(), log_bytes, log_region, iters, sink.as<uint32_t>());
        HB_CUDA(cudaEventRecord(e1));
        HB_CUDA(cudaEventSynchronize(e1));
        HB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *gbs = (double)iters * 32 * 32 / (ms * 1e-3) / 1e9;
    return HBFS_OK;
    HB_ENTRY_END
}

// Tuning: the L2's DRAM fetch granularity for this context (cudaLimitMaxL2FetchGranularity,
// 32..128 bytes).  previous (may be NULL) receives the value before the call; bytes < 0 only
// queries.
extern "C" int hbfs_l2_fetch_granularity(int bytes, int *previous) {
    HB_ENTRY_BEGIN
    using namespace hbfs;
    clear_error();
    size_t cur = 0;
    HB_CUDA(cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity));
    if (previous) *previous = (int)cur;
    if (bytes >= 0) {
        if (bytes > 128) return set_error(HBFS_EINVAL, "granularity must be <= 128 bytes");
        HB_CUDA(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes));
    }
    return HBFS_OK;
    HB_ENTRY_END
}

// ---- debugging aids (compute-sanitizer substitutes) ----

namespace hbfs {

namespace {
std::mutex g_guard_mu;
std::unordered_map<void *, size_t> &guards() {
    static std::unordered_map<void *, size_t> m;
    return m;
}
}  // namespace

bool guard_enabled() {
    static const bool on = [] {
        const char *e = getenv("HBFS_GUARD");
        return e && atoi(e) != 0;
    }();
    return on;
}

void guard_register(void *p, size_t bytes) {
    std::lock_guard<std::mutex> lk(g_guard_mu);
    guards()[p] = bytes;
}

void guard_unregister(void *p) {
    if (!guard_enabled()) return;
    std::lock_guard<std::mutex> lk(g_guard_mu);
    guards().erase(p);
}

}  // namespace hbfs

// Verify every live guard band: *clobbered = number of bands with a changed
// byte; *first_bytes = the allocation size of the first clobbered buffer.
extern "C" int hbfs_debug_guards(int *enabled, int64_t *checked, int64_t *clobbered, int64_t *first_bytes) {
    HB_ENTRY_BEGIN
    using namespace hbfs;
    clear_error();
    if (enabled) *enabled = guard_enabled() ? 1 : 0;
    int64_t nchk = 0, nbad = 0, first = -1;
    if (guard_enabled()) {
        HB_CUDA(cudaDeviceSynchronize());
        std::vector<unsigned char> h(kGuardBytes);
        std::lock_guard<std::mutex> lk(g_guard_mu);
        for (auto &kv : guards()) {
            HB_CUDA(cudaMemcpy(h.data(), static_cast<char *>(kv.first) + kv.second, kGuardBytes,
                               cudaMemcpyDeviceToHost));
            ++nchk;
            for (size_t i = 0; i < kGuardBytes; ++i)
                if (h[i] != kGuardByte) {
                    if (nbad == 0) first = (int64_t)kv.second;
                    ++nbad;
                    break;
                }
        }
    }
    if (checked) *checked = nchk;
    if (clobbered) *clobbered = nbad;
    if (first_bytes) *first_bytes = first;
    return HBFS_OK;
    HB_ENTRY_END
}

