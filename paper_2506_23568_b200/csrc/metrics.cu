// Image-quality metrics on device-resident volumes (reference: metrics.py:126-150
// psnr, metrics.py:170-190 max_intensity_projection), SURVEY §8(f) #4.
//
// PSNR is two streaming passes over the two volumes (HBM-bound): pass 1 the
// float64 sums T = sum |t|^2, C = sum conj(t) r, R = sum |r|^2 and max |r|;
// the host forms the least-squares scale s = C / T (np.vdot(tst, ref) /
// np.vdot(tst, tst)); pass 2 E = sum |s t - r|^2.  Both passes reduce
// per-CTA partials in a fixed order (deterministic for a given device).
// The MIP is a max-|v| reduction along one axis (float64 magnitudes of the
// complex samples) followed by the dB mapping onto [0, 1].
#include <cfloat>

#include "common.cuh"

namespace hhsar {

constexpr int MET_THREADS = 256;

template <typename C>
struct Cplx;
template <>
struct Cplx<float2> {
    __device__ static double re(float2 v) { return (double)v.x; }
    __device__ static double im(float2 v) { return (double)v.y; }
};
template <>
struct Cplx<double2> {
    __device__ static double re(double2 v) { return v.x; }
    __device__ static double im(double2 v) { return v.y; }
};

// |v|^2 in float64; maxima are taken on squares and the (monotone,
// correctly rounded) sqrt applied once to the result -- within 1 ulp of
// numpy's hypot for these magnitudes
template <typename C>
__device__ __forceinline__ double cabs2_d(C v) {
    const double a = Cplx<C>::re(v), b = Cplx<C>::im(v);
    return fma(a, a, b * b);
}

template <int N>
__device__ __forceinline__ void block_sum(double (&v)[N], double *s_part) {
#pragma unroll
    for (int k = 0; k < N; ++k)
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < N; ++k) s_part[k * (MET_THREADS / 32) + wid] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < N; ++k) {
        double a = 0.0;
        for (int w = 0; w < MET_THREADS / 32; ++w) a += s_part[k * (MET_THREADS / 32) + w];
        v[k] = a;
    }
}

// partial[b] = (T, C.re, C.im, R, max|r|) of CTA b's grid-stride share
template <typename C>
__global__ void __launch_bounds__(MET_THREADS)
volume_dot_kernel(const C *__restrict__ t, const C *__restrict__ r, int64_t n,
                  double *__restrict__ partial) {
    __shared__ double s_part[4 * MET_THREADS / 32];
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    double mx = 0.0;
#pragma unroll 4
    for (int64_t i = (int64_t)blockIdx.x * MET_THREADS + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * MET_THREADS) {
        const C a = t[i], b = r[i];
        const double ar = Cplx<C>::re(a), ai = Cplx<C>::im(a);
        const double br = Cplx<C>::re(b), bi = Cplx<C>::im(b);
        v[0] += ar * ar + ai * ai;  // same expression as C.re when r == t
        v[1] += ar * br + ai * bi;
        v[2] += ar * bi - ai * br;
        v[3] += br * br + bi * bi;
        mx = fmax(mx, fma(br, br, bi * bi));
    }
    block_sum(v, s_part);
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < MET_THREADS / 32; ++w) mx = fmax(mx, s_part[w]);
        double *p = partial + 5 * (int64_t)blockIdx.x;
        p[0] = v[0];
        p[1] = v[1];
        p[2] = v[2];
        p[3] = v[3];
        p[4] = sqrt(mx);
    }
}

// partial[b] = sum |s t - r|^2 over CTA b's share
template <typename C>
__global__ void __launch_bounds__(MET_THREADS)
volume_residual_kernel(const C *__restrict__ t, const C *__restrict__ r, int64_t n, double sr,
                       double si, double *__restrict__ partial) {
    __shared__ double s_part[MET_THREADS / 32];
    double v[1] = {0.0};
#pragma unroll 4
    for (int64_t i = (int64_t)blockIdx.x * MET_THREADS + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * MET_THREADS) {
        const C a = t[i], b = r[i];
        const double ar = Cplx<C>::re(a), ai = Cplx<C>::im(a);
        const double er = (ar * sr - ai * si) - Cplx<C>::re(b);
        const double ei = (ar * si + ai * sr) - Cplx<C>::im(b);
        v[0] += er * er + ei * ei;
    }
    block_sum(v, s_part);
    if (threadIdx.x == 0) partial[blockIdx.x] = v[0];
}

// out[k] = reduction over CTAs of partial[b * width + k] (max for k in
// max_mask): one warp per column, lanes take CTAs lane, lane + 32, ... and a
// fixed shuffle tree combines them (deterministic).
__global__ void reduce_partials_kernel(const double *__restrict__ partial, int nb, int width,
                                       unsigned max_mask, double *__restrict__ out) {
    const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (k >= width) return;
    const bool is_max = (max_mask >> k) & 1u;
    double a = 0.0;  // sums start at 0; maxima of magnitudes too
    for (int b = lane; b < nb; b += 32) {
        const double x = partial[(int64_t)b * width + k];
        a = is_max ? fmax(a, x) : a + x;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double y = __shfl_xor_sync(0xffffffffu, a, o);
        a = is_max ? fmax(a, y) : a + y;
    }
    if (lane == 0) out[k] = a;
}

// MIP: out[(a, b)] = max over the projected axis of |v|; dims (n0, n1, n2),
// the output keeps the two other axes in order.  Axis 2 (contiguous runs):
// one warp per output; axes 0/1: one thread per output, consecutive outputs
// read consecutive addresses.
template <typename C>
__global__ void mip_rows_kernel(const C *__restrict__ v, int64_t rows, int64_t n2,
                                double *__restrict__ out) {
    const int64_t o = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (o >= rows) return;  // warp-uniform
    const C *p = v + o * n2;
    double m = 0.0;
#pragma unroll 8
    for (int64_t k = lane; k < n2; k += 32) m = fmax(m, cabs2_d(p[k]));
    for (int s = 16; s > 0; s >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, s));
    if (lane == 0) out[o] = sqrt(m);
}

template <typename C>
__global__ void mip_strided_kernel(const C *__restrict__ v, int64_t n0, int64_t n1, int64_t n2,
                                   int axis, double *__restrict__ out) {
    const int64_t no = axis == 0 ? n1 * n2 : n0 * n2;
    const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= no) return;
    double m = 0.0;
    if (axis == 1) {  // out (i, k) = max_j v[i, j, k]
        const int64_t i = o / n2, k = o % n2;
        const C *p = v + i * n1 * n2 + k;
#pragma unroll 8
        for (int64_t j = 0; j < n1; ++j)
            m = fmax(m, cabs2_d(p[j * n2]));
    } else {  // out (j, k) = max_i v[i, j, k]
        const C *p = v + o;
#pragma unroll 8
        for (int64_t i = 0; i < n0; ++i)
            m = fmax(m, cabs2_d(p[i * n1 * n2]));
    }
    out[o] = sqrt(m);
}

// Grid-wide max of non-negative doubles: their bit patterns order like
// unsigned integers, so one atomicMax per CTA (order-independent, exact).
__global__ void max_kernel(const double *__restrict__ x, int64_t n,
                           unsigned long long *__restrict__ out_bits) {
    __shared__ double s[MET_THREADS / 32];
    double m = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * MET_THREADS + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * MET_THREADS)
        m = fmax(m, x[i]);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < MET_THREADS / 32; ++w) m = fmax(m, s[w]);
        atomicMax(out_bits, (unsigned long long)__double_as_longlong(m));
    }
}

// dB scaling relative to the peak, clipped at floor_db, mapped onto [0, 1]
// (metrics.py:180-190); an all-zero projection stays zero.
__global__ void mip_map_kernel(double *__restrict__ x, int64_t n, const double *__restrict__ peak,
                               double floor_db) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double p = peak[0];
    if (p == 0.0) {
        x[i] = 0.0;
        return;
    }
    const double db = fmax(20.0 * log10(x[i] / p), floor_db);  // log10(0) = -inf -> floor
    x[i] = (db - floor_db) / (-floor_db);
}

static int metric_blocks(int64_t n) {
    int64_t nb = (n + MET_THREADS - 1) / MET_THREADS;
    const int64_t cap = 8 * (int64_t)sm_count();
    return (int)(nb < cap ? (nb < 1 ? 1 : nb) : cap);
}

}  // namespace hhsar

using namespace hhsar;

extern "C" int hhsar_volume_dot(const void *test, const void *ref, int64_t n, int dtype,
                                double *out5, void *stream) {
    HHSAR_REQUIRE(n >= 0 && (dtype == 0 || dtype == 1) && out5, "volume_dot: bad arguments");
    cudaStream_t s = as_stream(stream);
    const int nb = metric_blocks(n);
    double *part = nullptr;
    if (cudaMallocAsync(&part, sizeof(double) * 5 * nb, s) != cudaSuccess)
        return set_error(HHSAR_ECUDA, "volume_dot: scratch allocation failed");
    if (dtype == 0)
        volume_dot_kernel<float2><<<nb, MET_THREADS, 0, s>>>(
            reinterpret_cast<const float2 *>(test), reinterpret_cast<const float2 *>(ref), n, part);
    else
        volume_dot_kernel<double2><<<nb, MET_THREADS, 0, s>>>(
            reinterpret_cast<const double2 *>(test), reinterpret_cast<const double2 *>(ref), n,
            part);
    reduce_partials_kernel<<<1, 5 * 32, 0, s>>>(part, nb, 5, 1u << 4, out5);
    cudaFreeAsync(part, s);
    return check_launch("volume_dot_kernel");
}

extern "C" int hhsar_volume_residual(const void *test, const void *ref, int64_t n, int dtype,
                                     double scale_re, double scale_im, double *out1,
                                     void *stream) {
    HHSAR_REQUIRE(n >= 0 && (dtype == 0 || dtype == 1) && out1, "volume_residual: bad arguments");
    cudaStream_t s = as_stream(stream);
    const int nb = metric_blocks(n);
    double *part = nullptr;
    if (cudaMallocAsync(&part, sizeof(double) * nb, s) != cudaSuccess)
        return set_error(HHSAR_ECUDA, "volume_residual: scratch allocation failed");
    if (dtype == 0)
        volume_residual_kernel<float2><<<nb, MET_THREADS, 0, s>>>(
            reinterpret_cast<const float2 *>(test), reinterpret_cast<const float2 *>(ref), n,
            scale_re, scale_im, part);
    else
        volume_residual_kernel<double2><<<nb, MET_THREADS, 0, s>>>(
            reinterpret_cast<const double2 *>(test), reinterpret_cast<const double2 *>(ref), n,
            scale_re, scale_im, part);
    reduce_partials_kernel<<<1, 32, 0, s>>>(part, nb, 1, 0u, out1);
    cudaFreeAsync(part, s);
    return check_launch("volume_residual_kernel");
}

extern "C" int hhsar_mip(const void *volume, const int64_t *dims, int dtype, int axis,
                         double floor_db, double *out, void *stream) {
    HHSAR_REQUIRE(dims && dims[0] > 0 && dims[1] > 0 && dims[2] > 0 && out,
                  "mip: bad dimensions");
    HHSAR_REQUIRE(dtype == 0 || dtype == 1, "mip: dtype must be 0 (complex64) or 1 (complex128)");
    HHSAR_REQUIRE(axis >= 0 && axis <= 2, "mip: axis index must be 0, 1, or 2");
    HHSAR_REQUIRE(floor_db < 0.0, "mip: floor must be below 0 dB");
    cudaStream_t s = as_stream(stream);
    const int64_t no = axis == 0 ? dims[1] * dims[2] : axis == 1 ? dims[0] * dims[2]
                                                                 : dims[0] * dims[1];
    const unsigned blocks = (unsigned)((no + MET_THREADS - 1) / MET_THREADS);
    const unsigned row_blocks = (unsigned)((no * 32 + MET_THREADS - 1) / MET_THREADS);
    if (axis == 2) {
        if (dtype == 0)
            mip_rows_kernel<float2><<<row_blocks, MET_THREADS, 0, s>>>(
                reinterpret_cast<const float2 *>(volume), no, dims[2], out);
        else
            mip_rows_kernel<double2><<<row_blocks, MET_THREADS, 0, s>>>(
                reinterpret_cast<const double2 *>(volume), no, dims[2], out);
    } else if (dtype == 0) {
        mip_strided_kernel<float2><<<blocks, MET_THREADS, 0, s>>>(
            reinterpret_cast<const float2 *>(volume), dims[0], dims[1], dims[2], axis, out);
    } else {
        mip_strided_kernel<double2><<<blocks, MET_THREADS, 0, s>>>(
            reinterpret_cast<const double2 *>(volume), dims[0], dims[1], dims[2], axis, out);
    }
    double *peak = nullptr;
    if (cudaMallocAsync(&peak, sizeof(double), s) != cudaSuccess)
        return set_error(HHSAR_ECUDA, "mip: scratch allocation failed");
    cudaMemsetAsync(peak, 0, sizeof(double), s);  // +0.0
    max_kernel<<<metric_blocks(no), MET_THREADS, 0, s>>>(
        out, no, reinterpret_cast<unsigned long long *>(peak));
    mip_map_kernel<<<blocks, MET_THREADS, 0, s>>>(out, no, peak, floor_db);
    cudaFreeAsync(peak, s);
    return check_launch("mip_rows_kernel / mip_strided_kernel");
}
