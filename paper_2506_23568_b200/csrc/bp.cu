// Backprojection gather kernels (reference: _kernels.py:44-110, bpa.py:144-176).
//
// One "unit" is one (voxel, element) pair: distance, delay-bin lookup with
// linear interpolation of the complex64 envelope, carrier phase exp(j 2 k_ref
// d) with explicit range reduction, complex accumulate.  FP32 + SFU bound;
// element positions are staged in shared memory per chunk and broadcast.
#include "common.cuh"

namespace hhsar {

constexpr int BP_THREADS = 256;
constexpr int BP_CHUNK = 512;   // elements staged per shared-memory pass
constexpr int CART_V = 4;       // voxels per thread along x
constexpr int CART_TZ = 64;     // tile: CART_V (x) x 4 (y) x 64 (z)
constexpr int CART_TY = BP_THREADS / CART_TZ;

struct BpConst {
    float inv_bin;   // 2 / (c * dt): metres -> delay-bin index
    float x0;        // t0 / dt
    float rev;       // k_ref / pi: metres -> carrier revolutions (2 k_ref d / 2 pi)
    float xmax;      // n_t - 1
    int n_t;
};

// One unit: returns false (and contributes nothing) when the delay is outside
// the profile window, exactly like the reference's skip-and-count.
__device__ __forceinline__ bool bp_unit(float d, const BpConst &k, const float2 *__restrict__ row,
                                        float2 &acc) {
    const float x = fmaf(d, k.inv_bin, -k.x0);
    if (!(x >= 0.f && x <= k.xmax)) return false;
    int i = min((int)x, k.n_t - 2);
    const float f = x - (float)i;
    const float2 v0 = __ldg(row + i), v1 = __ldg(row + i + 1);
    const float er = fmaf(f, v1.x - v0.x, v0.x), ei = fmaf(f, v1.y - v0.y, v0.y);
    // carrier exp(j k_ref c tau) = exp(j 2 pi * d k_ref / pi): reduce the
    // revolution count to [-0.5, 0.5] before the SFU sincos
    const float rv = d * k.rev;
    const float red = __fsub_rn(rv, rintf(rv));
    float s, c;
    __sincosf(6.283185307f * red, &s, &c);
    acc.x = fmaf(er, c, fmaf(-ei, s, acc.x));
    acc.y = fmaf(er, s, fmaf(ei, c, acc.y));
    return true;
}

// Full-aperture BPA over region_grid voxels, flattened index in [vb, ve).
__global__ void __launch_bounds__(BP_THREADS)
bpa_cartesian_kernel(double ox, double oy, double oz, double sx, double sy, double sz, int nx,
                     int ny, int nz, int64_t vb, int64_t ve, const float4 *__restrict__ el,
                     int m, const float2 *__restrict__ env, BpConst k,
                     float2 *__restrict__ out, int64_t *__restrict__ oow_total) {
    __shared__ float4 s_el[BP_CHUNK];
    // tile coordinates
    const int tiles_z = (nz + CART_TZ - 1) / CART_TZ;
    const int tiles_y = (ny + CART_TY - 1) / CART_TY;
    const int tiles_x = (nx + CART_V - 1) / CART_V;
    (void)tiles_x;
    const int tile = blockIdx.x;
    const int tz = tile % tiles_z, ty = (tile / tiles_z) % tiles_y, tx = tile / (tiles_z * tiles_y);
    const int iz = tz * CART_TZ + (threadIdx.x % CART_TZ);
    const int iy = ty * CART_TY + (threadIdx.x / CART_TZ);
    const int ix0 = tx * CART_V;
    // voxel coordinates exactly as numpy: origin + step * i (float64), then f32
    const float py = (float)__dadd_rn(oy, __dmul_rn(sy, (double)iy));
    const float pz = (float)__dadd_rn(oz, __dmul_rn(sz, (double)iz));
    float px[CART_V];
    bool live[CART_V];
    int64_t flat[CART_V];
#pragma unroll
    for (int v = 0; v < CART_V; ++v) {
        const int ix = ix0 + v;
        px[v] = (float)__dadd_rn(ox, __dmul_rn(sx, (double)ix));
        flat[v] = ((int64_t)ix * ny + iy) * nz + iz;
        live[v] = ix < nx && iy < ny && iz < nz && flat[v] >= vb && flat[v] < ve;
    }
    float2 acc[CART_V];
    unsigned bad = 0;
#pragma unroll
    for (int v = 0; v < CART_V; ++v) acc[v] = make_float2(0.f, 0.f);

    for (int c0 = 0; c0 < m; c0 += BP_CHUNK) {
        const int cn = min(BP_CHUNK, m - c0);
        __syncthreads();
        for (int j = threadIdx.x; j < cn; j += BP_THREADS) s_el[j] = el[c0 + j];
        __syncthreads();
        for (int j = 0; j < cn; ++j) {
            const float4 e = s_el[j];
            const float dy = py - e.y, dz = pz - e.z;
            const float dyz = fmaf(dy, dy, dz * dz);
            const float2 *row = env + (int64_t)(c0 + j) * k.n_t;
#pragma unroll
            for (int v = 0; v < CART_V; ++v) {
                const float dx = px[v] - e.x;
                const float d = sqrtf(fmaf(dx, dx, dyz));
                if (live[v]) bad += !bp_unit(d, k, row, acc[v]);
            }
        }
    }
#pragma unroll
    for (int v = 0; v < CART_V; ++v)
        if (live[v]) out[flat[v] - vb] = acc[v];
    if (bad) atomicAdd((unsigned long long *)oow_total, (unsigned long long)bad);
}

// Generic gather for arbitrary points (operator-level backproject_gather).
__global__ void __launch_bounds__(BP_THREADS)
bp_gather_kernel(const double *__restrict__ pts, int64_t n, const float4 *__restrict__ el, int m,
                 const float2 *__restrict__ env, BpConst k, float2 *__restrict__ out,
                 int64_t *__restrict__ oow) {
    __shared__ float4 s_el[BP_CHUNK];
    const int64_t p = (int64_t)blockIdx.x * BP_THREADS + threadIdx.x;
    const bool live = p < n;
    float px = 0.f, py = 0.f, pz = 0.f;
    if (live) {
        px = (float)pts[3 * p];
        py = (float)pts[3 * p + 1];
        pz = (float)pts[3 * p + 2];
    }
    float2 acc = make_float2(0.f, 0.f);
    int64_t bad = 0;
    for (int c0 = 0; c0 < m; c0 += BP_CHUNK) {
        const int cn = min(BP_CHUNK, m - c0);
        __syncthreads();
        for (int j = threadIdx.x; j < cn; j += BP_THREADS) s_el[j] = el[c0 + j];
        __syncthreads();
        if (live)
            for (int j = 0; j < cn; ++j) {
                const float4 e = s_el[j];
                const float dx = px - e.x, dy = py - e.y, dz = pz - e.z;
                const float d = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                bad += !bp_unit(d, k, env + (int64_t)(c0 + j) * k.n_t, acc);
            }
    }
    if (live) {
        out[p] = acc;
        oow[p] = bad;
    }
}

__global__ void el_to_f32x4(const double *__restrict__ el, int64_t m, float4 *__restrict__ o) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) o[i] = make_float4((float)el[3 * i], (float)el[3 * i + 1], (float)el[3 * i + 2], 0.f);
}

BpConst make_bp_const(int64_t n_t, double t0, double dt, double k_ref) {
    BpConst k;
    k.inv_bin = (float)(2.0 / (HHSAR_C_LIGHT * dt));
    k.x0 = (float)(t0 / dt);
    k.rev = (float)(k_ref / 3.141592653589793);
    k.xmax = (float)(n_t - 1);
    k.n_t = (int)n_t;
    return k;
}

}  // namespace hhsar

using namespace hhsar;

extern "C" int hhsar_bpa_cartesian(const double *origin, const double *step, const int64_t *dims,
                                   int64_t vox_begin, int64_t vox_end, const float *el_xyz,
                                   int64_t m, const void *envelopes, int64_t n_t, double t0,
                                   double dt, double k_ref, void *out, int64_t *oow_total,
                                   void *stream) {
    HHSAR_REQUIRE(dims[0] > 0 && dims[1] > 0 && dims[2] > 0, "bpa_cartesian: empty dims");
    HHSAR_REQUIRE(n_t >= 2, "bpa_cartesian: n_t must be >= 2");
    HHSAR_REQUIRE(m >= 0 && m < (1ll << 31), "bpa_cartesian: bad element count");
    const int64_t total = dims[0] * dims[1] * dims[2];
    if (vox_end < 0 || vox_end > total) vox_end = total;
    HHSAR_REQUIRE(vox_begin >= 0 && vox_begin <= vox_end, "bpa_cartesian: bad voxel range");
    if (vox_begin == vox_end) return HHSAR_OK;
    const int nx = (int)dims[0], ny = (int)dims[1], nz = (int)dims[2];
    const int64_t tiles = (int64_t)((nx + CART_V - 1) / CART_V) * ((ny + CART_TY - 1) / CART_TY) *
                          ((nz + CART_TZ - 1) / CART_TZ);
    cudaStream_t s = as_stream(stream);
    if (m == 0) {
        cudaMemsetAsync(out, 0, (vox_end - vox_begin) * sizeof(float2), s);
        return check_launch("bpa_cartesian memset");
    }
    bpa_cartesian_kernel<<<(unsigned)tiles, BP_THREADS, 0, s>>>(
        origin[0], origin[1], origin[2], step[0], step[1], step[2], nx, ny, nz, vox_begin,
        vox_end, reinterpret_cast<const float4 *>(el_xyz), (int)m,
        reinterpret_cast<const float2 *>(envelopes), make_bp_const(n_t, t0, dt, k_ref),
        reinterpret_cast<float2 *>(out), oow_total);
    return check_launch("bpa_cartesian_kernel");
}

extern "C" int hhsar_bp_gather(const double *points, int64_t n, const double *el_pos, int64_t m,
                               const void *envelopes, int64_t n_t, double t0, double dt,
                               double k_ref, void *out, int64_t *oow, void *stream) {
    HHSAR_REQUIRE(n >= 0 && m >= 0 && m < (1ll << 31), "bp_gather: bad sizes");
    HHSAR_REQUIRE(n_t >= 2, "bp_gather: n_t must be >= 2");
    if (n == 0) return HHSAR_OK;
    cudaStream_t s = as_stream(stream);
    if (m == 0) {
        cudaMemsetAsync(out, 0, n * sizeof(float2), s);
        cudaMemsetAsync(oow, 0, n * sizeof(int64_t), s);
        return check_launch("bp_gather memset");
    }
    float4 *el4 = nullptr;
    if (cudaMallocAsync(&el4, m * sizeof(float4), s) != cudaSuccess)
        return set_error(HHSAR_ECUDA, "bp_gather: allocation failed");
    el_to_f32x4<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(el_pos, m, el4);
    bp_gather_kernel<<<(unsigned)((n + BP_THREADS - 1) / BP_THREADS), BP_THREADS, 0, s>>>(
        points, n, el4, (int)m, reinterpret_cast<const float2 *>(envelopes),
        make_bp_const(n_t, t0, dt, k_ref), reinterpret_cast<float2 *>(out), oow);
    cudaFreeAsync(el4, s);
    return check_launch("bp_gather_kernel");
}
