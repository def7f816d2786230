// Range-compression helpers around the batched IDFT and the Born simulator
// (reference: rangecomp.py:61-101, simulator.py:41-69).
#include "common.cuh"

namespace hhsar {

__global__ void range_pad_kernel(const float2 *__restrict__ cube, int64_t n_el, int n_f, int n_t,
                                 float2 *__restrict__ spec) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_el * n_t) return;
    const int64_t e = idx / n_t;
    const int i = (int)(idx % n_t);
    spec[idx] = i < n_f ? cube[e * n_f + i] : make_float2(0.f, 0.f);
}

// envelopes = profiles * exp(j * a * (dt * i)), a = (k_min - k_ref) * c
// (rangecomp.py:94-96); float64 phase per bin, reduced before the SFU.
__global__ void range_demod_kernel(float2 *__restrict__ prof, int64_t n_el, int n_t, double a,
                                   double dt, float scale) {
    __shared__ float2 s_rot[1024];
    for (int c0 = 0; c0 < n_t; c0 += 1024) {
        const int cn = min(1024, n_t - c0);
        __syncthreads();
        for (int i = threadIdx.x; i < cn; i += blockDim.x) {
            const float2 r = cis_reduced(a * (dt * (double)(c0 + i)));
            s_rot[i] = make_float2(r.x * scale, r.y * scale);
        }
        __syncthreads();
        for (int64_t e = blockIdx.y; e < n_el; e += gridDim.y) {
            float2 *row = prof + e * n_t + c0;
            for (int i = threadIdx.x; i < cn; i += blockDim.x) row[i] = cmul(row[i], s_rot[i]);
        }
    }
}

// ---------------------------------------------------------------------------
// Fused range compression: zero-pad + unnormalised inverse DFT + demodulation
// in one pass over HBM (read the n_f-sample cube row once, write the n_t-bin
// envelope row once).  One CTA per element row; the row lives in shared
// memory (ping-pong) and goes through Stockham autosort passes (radix 4,
// one radix-2 pass when log2 n_t is odd).  Twiddles and the demodulation
// phases come from float64-computed tables of n_t entries (L1/L2 resident).
// ---------------------------------------------------------------------------
constexpr int RC_THREADS = 256;

__global__ void rc_tables_kernel(float2 *__restrict__ roots, float2 *__restrict__ demod, int n,
                                 double a, double dt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s, c;
    sincospi(2.0 * (double)i / (double)n, &s, &c);  // e^{+2 pi j i / n}: inverse DFT
    roots[i] = make_float2((float)c, (float)s);
    demod[i] = cis_reduced(a * (dt * (double)i));   // rangecomp.py:95-96
}

template <int LOGN>
__global__ void __launch_bounds__(RC_THREADS)
range_compress_kernel(const float2 *__restrict__ cube, int n_f, const float2 *__restrict__ roots,
                      const float2 *__restrict__ demod, float2 *__restrict__ out) {
    constexpr int N = 1 << LOGN;
    extern __shared__ float2 rc_smem[];
    float2 *in = rc_smem, *tmp = rc_smem + N;
    const int64_t row = blockIdx.x;
    const float2 *src = cube + row * n_f;
    for (int i = threadIdx.x; i < N; i += RC_THREADS)
        in[i] = i < n_f ? src[i] : make_float2(0.f, 0.f);
    __syncthreads();
    int ns = 1;
    if (LOGN & 1) {  // one radix-2 pass first
        for (int j = threadIdx.x; j < N / 2; j += RC_THREADS) {
            const float2 v0 = in[j], v1 = in[j + N / 2];
            tmp[2 * j] = make_float2(v0.x + v1.x, v0.y + v1.y);
            tmp[2 * j + 1] = make_float2(v0.x - v1.x, v0.y - v1.y);
        }
        __syncthreads();
        float2 *t = in;
        in = tmp;
        tmp = t;
        ns = 2;
    }
    for (; ns < N; ns *= 4) {
        for (int j = threadIdx.x; j < N / 4; j += RC_THREADS) {
            const int k = j & (ns - 1);              // j % ns
            const int tw = k * (N / (4 * ns));        // twiddle step in units of 2 pi / N
            float2 v0 = in[j], v1 = in[j + N / 4], v2 = in[j + N / 2], v3 = in[j + 3 * N / 4];
            v1 = cmul(v1, roots[tw]);
            v2 = cmul(v2, roots[2 * tw]);
            v3 = cmul(v3, roots[3 * tw]);
            // inverse radix-4 butterfly: y_r = sum_q v_q i^{q r}
            const float2 s02 = make_float2(v0.x + v2.x, v0.y + v2.y);
            const float2 d02 = make_float2(v0.x - v2.x, v0.y - v2.y);
            const float2 s13 = make_float2(v1.x + v3.x, v1.y + v3.y);
            const float2 d13 = make_float2(v1.x - v3.x, v1.y - v3.y);
            const int base = (j - k) * 4 + k;         // (j / ns) * ns * 4 + j % ns
            tmp[base] = make_float2(s02.x + s13.x, s02.y + s13.y);
            tmp[base + ns] = make_float2(d02.x - d13.y, d02.y + d13.x);      // + i d13
            tmp[base + 2 * ns] = make_float2(s02.x - s13.x, s02.y - s13.y);
            tmp[base + 3 * ns] = make_float2(d02.x + d13.y, d02.y - d13.x);  // - i d13
        }
        __syncthreads();
        float2 *t = in;
        in = tmp;
        tmp = t;
    }
    float2 *dst = out + row * N;
    for (int i = threadIdx.x; i < N; i += RC_THREADS) dst[i] = cmul(in[i], __ldg(demod + i));
}

template <int LOGN>
int launch_rc(const float2 *cube, int64_t n_el, int n_f, const float2 *roots, const float2 *demod,
              float2 *out, cudaStream_t s) {
    const size_t smem = 2 * sizeof(float2) * (1u << LOGN);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(range_compress_kernel<LOGN>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int64_t r0 = 0; r0 < n_el; r0 += 2147483647ll) {
        const int64_t rows = n_el - r0 < 2147483647ll ? n_el - r0 : 2147483647ll;
        range_compress_kernel<LOGN><<<(unsigned)rows, RC_THREADS, smem, s>>>(
            cube + r0 * n_f, n_f, roots, demod, out + r0 * ((int64_t)1 << LOGN));
    }
    return check_launch("range_compress_kernel");
}

// One CTA per element; threads over frequencies.  Scatterer distances are
// computed once per (element, scatterer) into shared memory, then each
// frequency thread accumulates refl * exp(-2j k d) with a float64 phase.
constexpr int SIM_CHUNK = 256;

__global__ void __launch_bounds__(256)
simulate_kernel(const double *__restrict__ el, const double *__restrict__ pos,
                const double *__restrict__ refl, int n_s, const double *__restrict__ k, int n_f,
                float2 *__restrict__ out) {
    __shared__ double s_d[SIM_CHUNK];
    __shared__ double2 s_r[SIM_CHUNK];
    const int64_t e = blockIdx.x;
    const double ex = el[3 * e], ey = el[3 * e + 1], ez = el[3 * e + 2];
    for (int f0 = 0; f0 < n_f; f0 += blockDim.x) {
        const int f = f0 + threadIdx.x;
        const double kf = f < n_f ? -2.0 * k[f] : 0.0;
        double ar = 0.0, ai = 0.0;
        for (int s0 = 0; s0 < n_s; s0 += SIM_CHUNK) {
            const int sn = min(SIM_CHUNK, n_s - s0);
            __syncthreads();
            for (int j = threadIdx.x; j < sn; j += blockDim.x) {
                const int q = s0 + j;
                const double dx = pos[3 * q] - ex, dy = pos[3 * q + 1] - ey, dz = pos[3 * q + 2] - ez;
                s_d[j] = sqrt(dx * dx + dy * dy + dz * dz);
                s_r[j] = make_double2(refl[2 * q], refl[2 * q + 1]);
            }
            __syncthreads();
            if (f < n_f)
                for (int j = 0; j < sn; ++j) {
                    const float2 c = cis_reduced(kf * s_d[j]);
                    ar += s_r[j].x * c.x - s_r[j].y * c.y;
                    ai += s_r[j].x * c.y + s_r[j].y * c.x;
                }
        }
        if (f < n_f) out[e * n_f + f] = make_float2((float)ar, (float)ai);
    }
}

}  // namespace hhsar

using namespace hhsar;

extern "C" int hhsar_range_pad(const void *cube, int64_t n_el, int64_t n_f, int64_t n_t,
                               void *spec, void *stream) {
    HHSAR_REQUIRE(n_el >= 0 && n_f >= 1 && n_t >= n_f, "range_pad: bad sizes");
    const int64_t total = n_el * n_t;
    if (total == 0) return HHSAR_OK;
    range_pad_kernel<<<(unsigned)((total + 255) / 256), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const float2 *>(cube), n_el, (int)n_f, (int)n_t,
        reinterpret_cast<float2 *>(spec));
    return check_launch("range_pad_kernel");
}

extern "C" int hhsar_range_demod(void *prof, int64_t n_el, int64_t n_t, double a, double dt,
                                 float scale, void *stream) {
    HHSAR_REQUIRE(n_el >= 0 && n_t >= 1, "range_demod: bad sizes");
    if (n_el == 0) return HHSAR_OK;
    const int64_t rows = n_el < 4 * sm_count() ? n_el : 4 * sm_count();
    dim3 grid(1, (unsigned)rows);
    range_demod_kernel<<<grid, 256, 0, as_stream(stream)>>>(reinterpret_cast<float2 *>(prof), n_el,
                                                            (int)n_t, a, dt, scale);
    return check_launch("range_demod_kernel");
}

extern "C" int hhsar_range_compress(const void *cube, int64_t n_el, int64_t n_f, int64_t n_t,
                                    double a, double dt, void *out, void *stream) {
    HHSAR_REQUIRE(n_el >= 0 && n_f >= 1 && n_t >= n_f, "range_compress: bad sizes");
    int logn = 0;
    while ((1ll << logn) < n_t) ++logn;
    HHSAR_REQUIRE((1ll << logn) == n_t && logn >= 4 && logn <= 13,
                  "range_compress: n_t must be a power of two in [16, 8192]");
    if (n_el == 0) return HHSAR_OK;
    cudaStream_t s = as_stream(stream);
    float2 *tables = nullptr;
    if (cudaMallocAsync(&tables, 2 * n_t * sizeof(float2), s) != cudaSuccess)
        return set_error(HHSAR_ECUDA, "range_compress: table allocation failed");
    rc_tables_kernel<<<(unsigned)((n_t + 255) / 256), 256, 0, s>>>(tables, tables + n_t, (int)n_t,
                                                                   a, dt);
    auto c = reinterpret_cast<const float2 *>(cube);
    auto o = reinterpret_cast<float2 *>(out);
    int rc = HHSAR_OK;
    switch (logn) {
        case 4: rc = launch_rc<4>(c, n_el, (int)n_f, tables, tables + n_t, o, s); break;
        case 5: rc = launch_rc<5>(c, n_el, (int)n_f, tables, tables + n_t, o, s); break;
        case 6: rc = launch_rc<6>(c, n_el, (int)n_f, tables, tables + n_t, o, s); break;
        case 7: rc = launch_rc<7>(c, n_el, (int)n_f, tables, tables + n_t, o, s); break;
        case 8: rc = launch_rc<8>(c, n_el, (int)n_f, tables, tables + n_t, o, s); break;
        case 9: rc = launch_rc<9>(c, n_el, (int)n_f, tables, tables + n_t, o, s); break;
        case 10: rc = launch_rc<10>(c, n_el, (int)n_f, tables, tables + n_t, o, s); break;
        case 11: rc = launch_rc<11>(c, n_el, (int)n_f, tables, tables + n_t, o, s); break;
        case 12: rc = launch_rc<12>(c, n_el, (int)n_f, tables, tables + n_t, o, s); break;
        default: rc = launch_rc<13>(c, n_el, (int)n_f, tables, tables + n_t, o, s); break;
    }
    cudaFreeAsync(tables, s);
    return rc;
}

extern "C" int hhsar_simulate(const double *el_pos, int64_t n_el, const double *pos,
                              const double *refl, int64_t n_s, const double *k, int64_t n_f,
                              void *out, void *stream) {
    HHSAR_REQUIRE(n_el >= 0 && n_s >= 0 && n_f >= 1 && n_el < (1ll << 31), "simulate: bad sizes");
    if (n_el == 0) return HHSAR_OK;
    simulate_kernel<<<(unsigned)n_el, 256, 0, as_stream(stream)>>>(
        el_pos, pos, refl, (int)n_s, k, (int)n_f, reinterpret_cast<float2 *>(out));
    return check_launch("simulate_kernel");
}
