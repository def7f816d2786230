// Shared device helpers for the sm_100a HHFFBPA / BPA kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hhsar_b200.h"

#define HHSAR_C_LIGHT 299792458.0

namespace hhsar {

// ---- status plumbing -------------------------------------------------------
int set_error(int code, const char *fmt, ...);
int check_launch(const char *what);

#define HHSAR_REQUIRE(cond, ...) \
    do { if (!(cond)) return ::hhsar::set_error(HHSAR_EINVAL, __VA_ARGS__); } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();                  // SM count of the current device (cached per device)
int current_device();
// Resident CTAs per SM of `kernel` at `threads` threads (cached per device
// and kernel, thread-safe).
int occupancy(const void *kernel, int threads, size_t smem = 0);
// High-priority non-blocking stream of the current device (created once,
// thread-safe); nullptr if it cannot be created.
cudaStream_t side_stream();

// ---- exact float64 arithmetic ----------------------------------------------
// numpy evaluates each ufunc separately with IEEE round-to-nearest and never
// fuses a multiply into an add.  The lattice bounds, counts and masks are
// integer decisions taken on float64 values, so the device code that
// reproduces them uses these wrappers to forbid FMA contraction.
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double xsqrt(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ double xsq(double a) { return __dmul_rn(a, a); }
__device__ __forceinline__ double xclip(double v, double lo, double hi) {
    return fmin(fmax(v, lo), hi);  // np.clip for finite lo <= hi
}

// Sum of distances from p to the four z'=0 vertices of the lateral box,
// ((daa + dab) + dba) + dbb  (spectrum.py:124-139), bit-exact with numpy.
__device__ __forceinline__ double corner_sum_exact(const double *ext, double x, double y,
                                                   double z) {
    const double z2 = xsq(z);
    const double xa = xsq(xsub(x, ext[0])), xb = xsq(xsub(x, ext[1]));
    const double ya = xsq(xsub(y, ext[2])), yb = xsq(xsub(y, ext[3]));
    const double daa = xsqrt(xadd(xadd(xa, ya), z2));
    const double dab = xsqrt(xadd(xadd(xa, yb), z2));
    const double dba = xsqrt(xadd(xadd(xb, ya), z2));
    const double dbb = xsqrt(xadd(xadd(xb, yb), z2));
    return xadd(xadd(xadd(daa, dab), dba), dbb);
}

__device__ __forceinline__ double box_gap_exact(const double *ext) {
    // 4.0 * dx ** 2 + 4.0 * dy ** 2   (spectrum.py:142-144)
    return xadd(xmul(4.0, xsq(xsub(ext[1], ext[0]))), xmul(4.0, xsq(xsub(ext[3], ext[2]))));
}

// llt_forward (spectrum.py:243-275), bit-exact; returns false outside the
// beta domain (rad <= gap * 1e-12).
__device__ __forceinline__ bool llt_exact(const double *ext, const hhsar_geom &g, double x,
                                          double y, double z, double *uvn) {
    const double x0 = xclip(x, ext[0], ext[1]);
    const double y0 = xclip(y, ext[2], ext[3]);
    const double z2 = xsq(z);
    const double dy0 = xsq(xsub(y, y0));
    const double u = xmul(g.c_uv, xsub(xsqrt(xadd(xadd(xsq(xsub(x, ext[0])), dy0), z2)),
                                       xsqrt(xadd(xadd(xsq(xsub(x, ext[1])), dy0), z2))));
    const double dx0 = xsq(xsub(x, x0));
    const double v = xmul(g.c_uv, xsub(xsqrt(xadd(xadd(dx0, xsq(xsub(y, ext[2]))), z2)),
                                       xsqrt(xadd(xadd(dx0, xsq(xsub(y, ext[3]))), z2))));
    const double r = corner_sum_exact(ext, x, y, z);
    const double gap = box_gap_exact(ext);
    const double rad = xsub(xmul(r, r), gap);
    uvn[0] = u;
    uvn[1] = v;
    uvn[2] = xsub(xmul(g.c_nhi, xsqrt(rad)), xmul(g.c_nlo, r));
    return !(rad <= xmul(gap, 1e-12));
}

// ---- single-MUFU fp32 approximations (ftz: no denormal rescaling around
// the SFU op, which the non-ftz forms add: 3 extra instructions each) ---------
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// ---- SFU-seeded float64 rsqrt / reciprocal --------------------------------------
// fp32 MUFU seed (relative error < 2^-22) refined by ONE float64 Newton step:
// relative error ~1.5 e0^2 < 1e-13.  Used where a float64 result feeds a
// tolerance far above 1e-13 (Newton residuals, merge coordinates and phases),
// never on the bit-exact lattice-metadata path.  Inputs must lie in the fp32
// normal range (squared distances of metres: fine).
__device__ __forceinline__ double rsqrt_d(double a) {
    double y;  // MUFU.RSQ64H seed (~2^-23), no fp32 round trip
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    const double e = fma(-(a * y), y, 1.0);
    return fma(0.5 * y, e, y);
}

__device__ __forceinline__ double rcp_d(double a) {
    double y;  // MUFU.RCP64H seed
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    return fma(y, fma(-a, y, 1.0), y);
}

// sqrt by one Heron step from the SFU rsqrt seed y: s0 = a y, s = s0 +
// (a - s0^2) y / 2 -- 4 float64 instructions, relative error ~2e-14
__device__ __forceinline__ double sqrt_d(double a) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    const double s0 = a * y;
    return fma(0.5 * y, fma(-s0, s0, a), s0);
}

// ---- fast float64 geometry for the merge stages ------------------------------
// Same formulas, FMA allowed (not on a bit-exactness path).
struct LltPhase {
    double u, v, n;   // compressed coordinates
    double phi;       // spatial downconversion phase, Eq. 30 (spectrum.py:229-240)
};

__device__ __forceinline__ LltPhase llt_phase(const double *ext, double gap, double c_uv,
                                              double c_nhi, double c_nlo, double k_min,
                                              double k_max, double x, double y, double z) {
    const double x0 = fmin(fmax(x, ext[0]), ext[1]);
    const double y0 = fmin(fmax(y, ext[2]), ext[3]);
    const double z2 = z * z;
    const double ax = x - ext[0], bx = x - ext[1], ay = y - ext[2], by = y - ext[3];
    const double xa = ax * ax, xb = bx * bx, ya = ay * ay, yb = by * by;
    const double dy0 = (y - y0) * (y - y0), dx0 = (x - x0) * (x - x0);
    LltPhase o;
    o.u = c_uv * (sqrt_d(xa + dy0 + z2) - sqrt_d(xb + dy0 + z2));
    o.v = c_uv * (sqrt_d(dx0 + ya + z2) - sqrt_d(dx0 + yb + z2));
    const double r = ((sqrt_d(xa + ya + z2) + sqrt_d(xa + yb + z2)) + sqrt_d(xb + ya + z2))
                     + sqrt_d(xb + yb + z2);
    const double sq = sqrt_d(r * r - gap);
    o.n = c_nhi * sq - c_nlo * r;
    o.phi = 0.25 * k_max * sq + 0.25 * k_min * r;
    return o;
}

__device__ __forceinline__ double sdc_phase_fast(const double *ext, double gap, double k_min,
                                                 double k_max, double x, double y, double z) {
    const double z2 = z * z;
    const double ax = x - ext[0], bx = x - ext[1], ay = y - ext[2], by = y - ext[3];
    const double xa = ax * ax, xb = bx * bx, ya = ay * ay, yb = by * by;
    const double r = ((sqrt_d(xa + ya + z2) + sqrt_d(xa + yb + z2)) + sqrt_d(xb + ya + z2))
                     + sqrt_d(xb + yb + z2);
    return 0.25 * k_max * sqrt_d(r * r - gap) + 0.25 * k_min * r;
}

// exp(j * phi) for a float64 phase of any size: explicit float64 reduction
// to [-pi, pi] followed by the fp32 SFU sincos.
__device__ __forceinline__ float2 cis_reduced(double phi) {
    const double two_pi = 6.283185307179586;
    const double inv_two_pi = 0.15915494309189535;
    const double red = fma(-two_pi, rint(phi * inv_two_pi), phi);
    float s, c;
    __sincosf((float)red, &s, &c);
    return make_float2(c, s);
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ void cfma(float2 &acc, float2 a, float2 b) {
    acc.x = fmaf(a.x, b.x, fmaf(-a.y, b.y, acc.x));
    acc.y = fmaf(a.x, b.y, fmaf(a.y, b.x, acc.y));
}

// ---- packed float32x2 (Blackwell FFMA2 / FADD2 / FMUL2) ---------------------
// Two independent fp32 lanes per instruction: halves the issue slots of the
// FMA-pipe work; a scalar operand is broadcast by ptxas (.F32 operand form).
struct f2x {
    unsigned long long r;
};
__device__ __forceinline__ f2x pk2(float lo, float hi) {
    f2x v;
    asm("mov.b64 %0, {%1, %2};" : "=l"(v.r) : "f"(lo), "f"(hi));
    return v;
}
__device__ __forceinline__ f2x bc2(float a) { return pk2(a, a); }
__device__ __forceinline__ float lo2(f2x v) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v.r));
    return a;
}
__device__ __forceinline__ float hi2(f2x v) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v.r));
    return b;
}
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) {
    f2x d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d.r) : "l"(a.r), "l"(b.r), "l"(c.r));
    return d;
}
__device__ __forceinline__ f2x add2(f2x a, f2x b) {
    f2x d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d.r) : "l"(a.r), "l"(b.r));
    return d;
}
__device__ __forceinline__ f2x add2_rm(f2x a, f2x b) {  // round toward -inf
    f2x d;
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(d.r) : "l"(a.r), "l"(b.r));
    return d;
}
__device__ __forceinline__ f2x sub2(f2x a, f2x b) {
    f2x d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d.r) : "l"(a.r), "l"(b.r));
    return d;
}
__device__ __forceinline__ f2x mul2(f2x a, f2x b) {
    f2x d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d.r) : "l"(a.r), "l"(b.r));
    return d;
}

// Keys cubic convolution weights, a = -1/2 (_kernels.py:192-200).
__device__ __forceinline__ void keys_weights(float f, float w[4]) {
    w[0] = ((-0.5f * f + 1.0f) * f - 0.5f) * f;
    w[1] = (1.5f * f - 2.5f) * f * f + 1.0f;
    w[2] = ((-1.5f * f + 2.0f) * f + 0.5f) * f;
    w[3] = (0.5f * f - 0.5f) * f * f;
}

// Lattice interpolation with the reference's hull rules (_kernels.py:117-189):
// linear needs every coordinate in [0, n-1] (base clamped to n-2), cubic in
// [1, n-2] (base clamped to n-3); outside -> ok = false, value 0.
// vals is [nu][nv][nn] complex64.  TU: type of the u, v coordinates (double
// on the API path, float inside the merge kernels); n is always double.
template <int KERNEL, typename TU = double>
__device__ __forceinline__ bool lattice_sample(const float2 *__restrict__ vals, int nu, int nv,
                                               int nn, TU cu, TU cv, double cn, float2 &out) {
    out = make_float2(0.f, 0.f);
    if (KERNEL == 0) {
        if (!(cu >= TU(0) && cu <= TU(nu - 1) && cv >= TU(0) && cv <= TU(nv - 1) && cn >= 0.0 &&
              cn <= nn - 1))
            return false;
        int iu = min((int)cu, nu - 2), iv = min((int)cv, nv - 2), iw = min((int)cn, nn - 2);
        const float fu = (float)(cu - iu), fv = (float)(cv - iv), fn = (float)(cn - iw);
        const float2 *b = vals + ((int64_t)iu * nv + iv) * nn + iw;
        const int64_t su = (int64_t)nv * nn;
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const float wa = a ? fu : 1.f - fu;
#pragma unroll
            for (int bb = 0; bb < 2; ++bb) {
                const float wb = bb ? fv : 1.f - fv;
                const float2 *row = b + a * su + bb * nn;
                const float2 v0 = __ldg(row), v1 = __ldg(row + 1);
                const float w0 = wa * wb * (1.f - fn), w1 = wa * wb * fn;
                acc.x = fmaf(v0.x, w0, fmaf(v1.x, w1, acc.x));
                acc.y = fmaf(v0.y, w0, fmaf(v1.y, w1, acc.y));
            }
        }
        out = acc;
        return true;
    } else {
        if (!(cu >= TU(1) && cu <= TU(nu - 2) && cv >= TU(1) && cv <= TU(nv - 2) && cn >= 1.0 &&
              cn <= nn - 2))
            return false;
        int iu = min((int)cu, nu - 3), iv = min((int)cv, nv - 3), iw = min((int)cn, nn - 3);
        float wu[4], wv[4], wn[4];
        keys_weights((float)(cu - iu), wu);
        keys_weights((float)(cv - iv), wv);
        keys_weights((float)(cn - iw), wn);
        const int64_t su = (int64_t)nv * nn;
        const float2 *b = vals + ((int64_t)(iu - 1) * nv + (iv - 1)) * nn + (iw - 1);
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                const float2 *row = b + a * su + bb * nn;
                const float w = wu[a] * wv[bb];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float2 v = __ldg(row + c);
                    acc.x = fmaf(v.x, w * wn[c], acc.x);
                    acc.y = fmaf(v.y, w * wn[c], acc.y);
                }
            }
        out = acc;
        return true;
    }
}

// Warp-aggregated counter increment: lanes that target the same counter are
// grouped (__match_any_sync), reduced, and the group leader adds once.
__device__ __forceinline__ void warp_add(int64_t *ctr, unsigned v) {
    const unsigned group = __match_any_sync(__activemask(), (unsigned long long)ctr);
    const unsigned s = __reduce_add_sync(group, v);
    if ((threadIdx.x & 31) == (unsigned)(__ffs(group) - 1) && s)
        atomicAdd((unsigned long long *)ctr, (unsigned long long)s);
}

// leaf2.cu: compacted point-list level-1 backprojection (hhsar_leaf_bp)
int launch_leaf_points(const hhsar_grid_desc *grids, int64_t n_grids, int64_t max_points,
                       int64_t pool_begin, int64_t pool_end, const double *positions,
                       const uint8_t *valid, const float4 *el, const float2 *env, int64_t n_t,
                       double t0, double dt, double k_ref, const hhsar_geom &g, int downconvert,
                       float2 *values, int64_t *oow_total, cudaStream_t s);

}  // namespace hhsar
