// Status plumbing shared by every C-ABI entry point.
#include <cstdarg>
#include <cstdio>

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

int sm_count() {
    static int cached = 0;
    if (!cached) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        if (cached <= 0) cached = 148;
        // Scratch buffers come from the stream-ordered pool (cudaMallocAsync);
        // keep freed blocks cached instead of returning them to the driver at
        // every synchronisation (threshold 0 by default), so repeated
        // reconstructions do not pay a cudaMalloc per call.
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    return cached;
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
