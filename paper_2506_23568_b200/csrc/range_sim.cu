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

extern "C" int hhsar_simulate(const double *el_pos, int64_t n_el, const double *pos,
                              const double *refl, int64_t n_s, const double *k, int64_t n_f,
                              void *out, void *stream) {
    HHSAR_REQUIRE(n_el >= 0 && n_s >= 0 && n_f >= 1 && n_el < (1ll << 31), "simulate: bad sizes");
    if (n_el == 0) return HHSAR_OK;
    simulate_kernel<<<(unsigned)n_el, 256, 0, as_stream(stream)>>>(
        el_pos, pos, refl, (int)n_s, k, (int)n_f, reinterpret_cast<float2 *>(out));
    return check_launch("simulate_kernel");
}
