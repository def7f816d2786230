// Status plumbing shared by every C-ABI entry point.
#include <cstdarg>
#include <cstdio>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

namespace hhsar {

static thread_local char g_err[512] = "";

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

int check_launch(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(HHSAR_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return HHSAR_OK;
}

// Per-device caches (SM count, occupancy, side streams).  They are the
// library's only process-wide state besides the thread-local error string;
// each entry is created once under a mutex and keyed by the calling thread's
// current device, so several host threads and several GPUs can share the
// library.
namespace {
constexpr int MAX_DEVICES = 64;
std::mutex g_cache_mutex;
int g_sm_count[MAX_DEVICES] = {};
std::map<std::pair<int, const void *>, int> g_occupancy;
cudaStream_t g_side_stream[MAX_DEVICES] = {};
}  // namespace

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

int sm_count() {
    const int dev = current_device();
    if (dev >= 0 && dev < MAX_DEVICES) {
        std::lock_guard<std::mutex> lock(g_cache_mutex);
        int &cached = g_sm_count[dev];
        if (!cached) {
            cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
            if (cached <= 0) cached = 148;
            // Scratch buffers come from the stream-ordered pool
            // (cudaMallocAsync); keep freed blocks cached instead of returning
            // them to the driver at every synchronisation (threshold 0 by
            // default), so repeated reconstructions do not pay a cudaMalloc
            // per call.
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t keep = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
        }
        return cached;
    }
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

int occupancy(const void *kernel, int threads, size_t smem) {
    const int dev = current_device();
    const auto key = std::make_pair(dev, kernel);
    {
        std::lock_guard<std::mutex> lock(g_cache_mutex);
        auto it = g_occupancy.find(key);
        if (it != g_occupancy.end()) return it->second;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    if (per_sm <= 0) per_sm = 1;
    std::lock_guard<std::mutex> lock(g_cache_mutex);
    g_occupancy[key] = per_sm;
    return per_sm;
}

cudaStream_t side_stream() {
    const int dev = current_device();
    if (dev < 0 || dev >= MAX_DEVICES) return nullptr;
    std::lock_guard<std::mutex> lock(g_cache_mutex);
    cudaStream_t &s = g_side_stream[dev];
    if (!s) {
        int lo = 0, hi = 0;  // highest priority: must not queue behind bulk CTAs
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi) != cudaSuccess) s = nullptr;
    }
    return s;
}

}  // namespace hhsar

extern "C" const char *hhsar_last_error(void) { return hhsar::g_err; }
extern "C" int hhsar_version(void) { return 1; }
extern "C" int hhsar_device_sm_count(void) { return hhsar::sm_count(); }

// ABI self-description for the host binding: struct sizes and field offsets
// the Python side checks its numpy mirrors against (no GPU needed).
#include <cstddef>
extern "C" int hhsar_abi_layout(int64_t *out, int n) {
    const int64_t v[] = {
        (int64_t)sizeof(hhsar_geom),
        (int64_t)sizeof(hhsar_grid_desc),
        (int64_t)offsetof(hhsar_geom, window_hi),
        (int64_t)offsetof(hhsar_geom, pad),
        (int64_t)offsetof(hhsar_grid_desc, dims),
        (int64_t)offsetof(hhsar_grid_desc, is_leaf),
        (int64_t)offsetof(hhsar_grid_desc, start),
        (int64_t)offsetof(hhsar_grid_desc, offset),
        (int64_t)offsetof(hhsar_grid_desc, col_offset),
    };
    const int k = (int)(sizeof v / sizeof v[0]);
    for (int i = 0; i < n && i < k; ++i) out[i] = v[i];
    return k;
}
