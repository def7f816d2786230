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

// Register-resident inverse DFTs (y_k = sum_n x_n e^{+2 pi i n k / R}), built
// as radix-2 splits down to the radix-4 butterfly; fully unrolled.
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// e^{+2 pi i q / R} for R in {8, 16}, q < R/2 (literal constants once unrolled)
template <int R>
__device__ __forceinline__ float2 root_of_unity(int q) {
    constexpr float c1 = 0.92387953251128674f, s1 = 0.38268343236508977f;
    constexpr float r2 = 0.70710678118654752f;
    if constexpr (R == 8) {
        switch (q) {
            case 0: return make_float2(1.f, 0.f);
            case 1: return make_float2(r2, r2);
            case 2: return make_float2(0.f, 1.f);
            default: return make_float2(-r2, r2);
        }
    } else {
        switch (q) {
            case 0: return make_float2(1.f, 0.f);
            case 1: return make_float2(c1, s1);
            case 2: return make_float2(r2, r2);
            case 3: return make_float2(s1, c1);
            case 4: return make_float2(0.f, 1.f);
            case 5: return make_float2(-s1, c1);
            case 6: return make_float2(-r2, r2);
            default: return make_float2(-c1, s1);
        }
    }
}

template <int R>
__device__ __forceinline__ void idft(float2 (&v)[R]) {
    if constexpr (R == 1) {
        return;
    } else if constexpr (R == 2) {
        const float2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    } else if constexpr (R == 4) {
        const float2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
        const float2 s13 = cadd(v[1], v[3]), d13 = csub(v[1], v[3]);
        v[0] = cadd(s02, s13);
        v[1] = make_float2(d02.x - d13.y, d02.y + d13.x);  // d02 + i d13
        v[2] = csub(s02, s13);
        v[3] = make_float2(d02.x + d13.y, d02.y - d13.x);  // d02 - i d13
    } else {
        constexpr int H = R / 2;
        float2 e[H], o[H];
#pragma unroll
        for (int q = 0; q < H; ++q) {
            e[q] = v[2 * q];
            o[q] = v[2 * q + 1];
        }
        idft<H>(e);
        idft<H>(o);
#pragma unroll
        for (int q = 0; q < H; ++q) {
            const float2 t = cmul(o[q], root_of_unity<R>(q));
            v[q] = cadd(e[q], t);
            v[q + H] = csub(e[q], t);
        }
    }
}

__device__ __forceinline__ int rc_pad(int i) { return i + (i >> 4); }  // breaks stride-16 bank conflicts

// One Stockham pass of radix R on the rows held in shared memory (or read
// from / written to global memory on the first / last pass).
template <int N, int R, bool FIRST, bool LAST>
__device__ __forceinline__ void rc_pass(int j, int ns, float2 *buf, const float2 *__restrict__ src,
                                        int n_f, bool live, const float2 *__restrict__ roots,
                                        const float2 *__restrict__ demod, float2 *__restrict__ dst) {
    float2 v[R];
    const int k = j & (ns - 1);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = j + r * (N / R);
        if (FIRST)
            v[r] = (live && i < n_f) ? __ldg(src + i) : make_float2(0.f, 0.f);
        else
            v[r] = buf[rc_pad(i)];
    }
    if (!FIRST) {
        const int t = k * (N / (ns * R));  // twiddle exponent step, units of 2 pi / N
        // w^1, w^2, w^4, w^8 from the float64-accurate table, the other powers
        // by products (<= 3 roundings): 4 loads instead of R - 1
        float2 w[R];
        w[1] = __ldg(roots + t);
        if (R > 2) w[2] = __ldg(roots + 2 * t);
        if (R > 4) w[4] = __ldg(roots + 4 * t);
        if (R > 8) w[8] = __ldg(roots + 8 * t);
#pragma unroll
        for (int r = 3; r < R; ++r) {
            const int hi = (r & 8) ? 8 : (r & 4) ? 4 : 2;  // highest power-of-two <= r
            if (r != hi) w[r] = cmul(w[hi], w[r - hi]);
        }
#pragma unroll
        for (int r = 1; r < R; ++r) v[r] = cmul(v[r], w[r]);
    }
    idft<R>(v);
    if (LAST) {
        // ns * R == N: j < ns, outputs land at j + r * N / R (coalesced)
        if (live) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int i = j + r * (N / R);
                dst[i] = cmul(v[r], __ldg(demod + i));
            }
        }
    } else {
        __syncthreads();  // every read of this pass precedes any write
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) buf[rc_pad(base + r * ns)] = v[r];
        __syncthreads();
    }
}

template <int LOGN>
struct RcShape {
    static constexpr int N = 1 << LOGN;
    static constexpr int T = N >= 16 ? N / 16 : 1;       // threads per row
    static constexpr int ROWS = T >= 256 ? 1 : 256 / T;  // rows per CTA
    static constexpr int NP = N + N / 16;                // padded row in smem
    static constexpr int REM = LOGN % 4;                 // radix 2^REM first pass
};

template <int LOGN>
__global__ void __launch_bounds__(RcShape<LOGN>::T * RcShape<LOGN>::ROWS,
                                  RcShape<LOGN>::T * RcShape<LOGN>::ROWS >= 512 ? 2 : 4)
range_compress_kernel(const float2 *__restrict__ cube, int64_t n_el, int n_f,
                      const float2 *__restrict__ roots, const float2 *__restrict__ demod,
                      float2 *__restrict__ out) {
    using S = RcShape<LOGN>;
    constexpr int N = S::N, T = S::T;
    extern __shared__ float2 rc_smem[];
    const int tx = threadIdx.x % T, ty = threadIdx.x / T;
    const int64_t row = (int64_t)blockIdx.x * S::ROWS + ty;
    const bool live = row < n_el;
    float2 *buf = rc_smem + ty * S::NP;
    const float2 *src = cube + (live ? row : 0) * n_f;
    float2 *dst = out + row * N;
    constexpr int P16 = LOGN / 4;  // radix-16 passes
    int ns = 1;
    if constexpr (S::REM > 0) {
        constexpr int R0 = 1 << S::REM;
#pragma unroll
        for (int m = 0; m < 16 / R0; ++m)  // N/R0 butterflies over T = N/16 threads
            if constexpr (P16 == 0) {
                rc_pass<N, R0, true, true>(tx + m * T, 1, buf, src, n_f, live, roots, demod, dst);
            } else {
                // first pass: butterflies j, stores without the trailing sync
                const int j = tx + m * T;
                float2 v[R0];
#pragma unroll
                for (int r = 0; r < R0; ++r) {
                    const int i = j + r * (N / R0);
                    v[r] = (live && i < n_f) ? __ldg(src + i) : make_float2(0.f, 0.f);
                }
                idft<R0>(v);
#pragma unroll
                for (int r = 0; r < R0; ++r) buf[rc_pad(j * R0 + r)] = v[r];
            }
        ns = R0;
        if constexpr (P16 > 0) __syncthreads();
    }
#pragma unroll
    for (int p = 0; p < P16; ++p) {
        const bool first = S::REM == 0 && p == 0, last = p == P16 - 1;
        if (first && last)
            rc_pass<N, 16, true, true>(tx, ns, buf, src, n_f, live, roots, demod, dst);
        else if (first)
            rc_pass<N, 16, true, false>(tx, ns, buf, src, n_f, live, roots, demod, dst);
        else if (last)
            rc_pass<N, 16, false, true>(tx, ns, buf, src, n_f, live, roots, demod, dst);
        else
            rc_pass<N, 16, false, false>(tx, ns, buf, src, n_f, live, roots, demod, dst);
        ns *= 16;
    }
}

template <int LOGN>
int launch_rc(const float2 *cube, int64_t n_el, int n_f, const float2 *roots, const float2 *demod,
              float2 *out, cudaStream_t s) {
    using S = RcShape<LOGN>;
    const size_t smem = sizeof(float2) * S::NP * S::ROWS;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(range_compress_kernel<LOGN>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t blocks = (n_el + S::ROWS - 1) / S::ROWS;
    for (int64_t b0 = 0; b0 < blocks; b0 += 2147483647ll) {
        const int64_t nb = blocks - b0 < 2147483647ll ? blocks - b0 : 2147483647ll;
        const int64_t r0 = b0 * S::ROWS;
        range_compress_kernel<LOGN><<<(unsigned)nb, S::T * S::ROWS, smem, s>>>(
            cube + r0 * n_f, n_el - r0, n_f, roots, demod, out + r0 * (int64_t)S::N);
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
