// Level-1 subimages, point-list form (reference: ffbp.py:310-348).
//
// 1. compact_leaf_kernel: per leaf grid, an ordered list of its valid
//    lattice points (block scan) in n-major order, so a CTA's points lie in a
//    thin range shell around the leaf's subaperture.
// 2. leaf_points_kernel: CTA = (leaf, chunk of 256 x P compacted points).
//    Same unit as the Cartesian BPA tile kernel: per element a delay window
//    of TW bins is staged in shared memory, bounded by the triangle
//    inequality |p - e| in [|p - c| - |e - c|, |p - c| + |e - c|] around the
//    leaf centre c over the chunk's points (TW = 32 ... 256 chosen per CTA
//    from the shell thickness and the leaf's element box); the window is
//    pre-rotated by the carrier, points are processed in pairs with packed
//    fp32x2 arithmetic; elements whose window does not fit take a checked
//    global-gather path (reference skip-and-count semantics).  Epilogue:
//    spatial downconversion exp(-j Phi_leaf(pos)) in float64, store to the
//    point's lattice slot (masked slots are zeroed beforehand).
#include "common.cuh"

namespace hhsar {

constexpr int LP_THREADS = 256;  // compact_leaf_kernel
#ifndef HHSAR_LEAF_THREADS
#define HHSAR_LEAF_THREADS 256
#endif
constexpr int LPT = HHSAR_LEAF_THREADS;  // leaf_points_kernel CTA (P points per thread)
constexpr int LPT_MINB = 1536 / LPT;     // CTAs per SM at 40 registers
constexpr float LP_MAGIC = 12582912.0f;
constexpr unsigned LP_MAGIC_BITS = 0x4B400000u;

struct LeafFast {
    float inv_bin, x0, xmax, cbin, kfrac, alpha, rev;
    int n_t;
    double alpha_d, kc_t0;
};

__global__ void __launch_bounds__(LP_THREADS)
compact_leaf_kernel(const hhsar_grid_desc *__restrict__ grids, const uint8_t *__restrict__ valid,
                    int32_t *__restrict__ idx, int32_t *__restrict__ cnt) {
    __shared__ int s_warp[LP_THREADS / 32];
    const hhsar_grid_desc &D = grids[blockIdx.x];
    const int nuv = D.dims[0] * D.dims[1], nn = D.dims[2];
    const int npts = nuv * nn;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int running = 0;
    for (int c0 = 0; c0 < npts; c0 += LP_THREADS) {
        // enumerate n-major: a chunk of the list is one or two n layers, i.e.
        // a thin shell of range around the leaf (tight delay windows)
        const int j = c0 + threadIdx.x;
        const int layer = j / nuv;
        const int i = (j - layer * nuv) * nn + layer;
        const bool f = j < npts && valid[D.offset + i];
        const unsigned ball = __ballot_sync(0xffffffffu, f);
        if (lane == 0) s_warp[wid] = __popc(ball);
        __syncthreads();
        int before = 0, total = 0;
        for (int q = 0; q < LP_THREADS / 32; ++q) {
            before += q < wid ? s_warp[q] : 0;
            total += s_warp[q];
        }
        if (f) idx[D.offset + running + before + __popc(ball & ((1u << lane) - 1u))] = i;
        running += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) cnt[blockIdx.x] = running;
}


// Carrier rotation per delay bin, exp(j k_ref c (t0 + dt bin)), float64 phase
// reduced then rounded once: shared by every element's window staging.
__global__ void leaf_rot_kernel(float2 *__restrict__ rot, int n_t, double kc_t0, double alpha_d) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_t) rot[i] = cis_reduced(kc_t0 + alpha_d * (double)i);
}

__device__ __forceinline__ float lp_sqrt(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

template <int P>
__global__ void __launch_bounds__(LPT, LPT_MINB)  // 1,536 threads per SM (40 registers)
leaf_points_kernel(const hhsar_grid_desc *__restrict__ grids, int chunks,
                   const int32_t *__restrict__ idx, const int32_t *__restrict__ cnt,
                   const double *__restrict__ positions, const float4 *__restrict__ el,
                   const float2 *__restrict__ env, const float2 *__restrict__ rot, LeafFast k,
                   hhsar_geom g, int downconvert, float2 *__restrict__ values,
                   int64_t *__restrict__ oow_total) {
    static_assert(P % 2 == 0, "points are processed in pairs");
    constexpr int WIN = 2048;  // staged window bins per pass: 32 KB
    __shared__ float4 s_env[WIN];
    __shared__ float4 s_el[WIN / 32];
    __shared__ int s_lo[WIN / 32];
    __shared__ int64_t s_row[WIN / 32];
    __shared__ float s_box[2][LPT / 32];
    const int gi = blockIdx.x / chunks, chunk = blockIdx.x % chunks;
    const hhsar_grid_desc &D = grids[gi];
    const int n = cnt[gi];
    const int p0 = chunk * LPT * P;
    if (p0 >= n) return;  // block-uniform
    const int t = threadIdx.x;
    // my points: P consecutive list entries per thread, so a partial last
    // chunk leaves whole warps without points (they skip the unit loop)
    float px[P], py[P], pz[P];
    int lat[P];
    // leaf centre (element bbox midpoint) and the chunk's range shell around it
    const float cx = (float)(0.5 * (D.box[0] + D.box[3])), cy = (float)(0.5 * (D.box[1] + D.box[4]));
    const float cz = (float)(0.5 * (D.box[2] + D.box[5]));
    float dmin = 3e38f, dmax = 0.f;
#pragma unroll
    for (int q = 0; q < P; ++q) {
        const int li = p0 + P * t + q;
        lat[q] = li < n ? idx[D.offset + li] : -1;
        const int src = lat[q] >= 0 ? lat[q] : idx[D.offset + p0];  // dead lanes mirror a live point
        const double *pp = positions + 3 * (D.offset + src);
        px[q] = (float)pp[0];
        py[q] = (float)pp[1];
        pz[q] = (float)pp[2];
        const float ex = px[q] - cx, ey = py[q] - cy, ez = pz[q] - cz;
        const float dc = sqrtf(fmaf(ex, ex, fmaf(ey, ey, ez * ez)));
        dmin = fminf(dmin, dc);
        dmax = fmaxf(dmax, dc);
    }
    const bool warp_live = __any_sync(0xffffffffu, lat[0] >= 0);
    for (int o = 16; o > 0; o >>= 1) {
        dmin = fminf(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
        dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    if ((t & 31) == 0) {
        s_box[0][t >> 5] = dmin;
        s_box[1][t >> 5] = dmax;
    }
    __syncthreads();
    dmin = s_box[0][0];
    dmax = s_box[1][0];
    for (int w = 1; w < LPT / 32; ++w) {
        dmin = fminf(dmin, s_box[0][w]);
        dmax = fmaxf(dmax, s_box[1][w]);
    }
    // window width for this chunk (block-uniform): the widest window any of
    // the leaf's elements needs (same bounds as the staging below)
    int need = 0;
    for (int64_t j = t; j < D.stop - D.start; j += LPT) {
        const float4 e = el[D.start + j];
        const float ex = e.x - cx, ey = e.y - cy, ez = e.z - cz;
        const float re = sqrtf(fmaf(ex, ex, fmaf(ey, ey, ez * ez)));
        const float xlo = fmaxf(dmin - re, 0.f) * k.inv_bin - k.x0;
        const float xhi = (dmax + re) * k.inv_bin - k.x0;
        if (xlo >= 1.f && xhi <= k.xmax - 2.f)
            need = max(need, min((int)floorf(xhi) + 2, k.n_t - 1) - max((int)floorf(xlo) - 2, 0) + 1);
    }
    need = __reduce_max_sync(0xffffffffu, need);
    __syncthreads();  // s_box reads above are done
    if ((t & 31) == 0) s_box[0][t >> 5] = __int_as_float(need);
    __syncthreads();
    for (int w = 0; w < LPT / 32; ++w) need = max(need, __float_as_int(s_box[0][w]));
    const int lw = need <= 32 ? 5 : need <= 64 ? 6 : need <= 128 ? 7 : 8;  // log2 TW
    const int TW = 1 << lw, LP_CHUNK = WIN >> lw;
    f2x pa[P], pb[P];
#pragma unroll
    for (int q = 0; q < P; ++q) pa[q] = pb[q] = pk2(0.f, 0.f);
    unsigned bad = 0;
    const int64_t e0 = D.start, m = D.stop - D.start;
    for (int64_t c0 = 0; c0 < m; c0 += LP_CHUNK) {
        const int cn = (int)min((int64_t)LP_CHUNK, m - c0);
        __syncthreads();
        int el_fast = 1;
        if (t < cn) {
            const float4 e = el[e0 + c0 + t];
            const float ex = e.x - cx, ey = e.y - cy, ez = e.z - cz;
            const float re = sqrtf(fmaf(ex, ex, fmaf(ey, ey, ez * ez)));
            const float xlo = fmaxf(dmin - re, 0.f) * k.inv_bin - k.x0;
            const float xhi = (dmax + re) * k.inv_bin - k.x0;
            const int lo = max((int)floorf(xlo) - 2, 0);
            const int hi = min((int)floorf(xhi) + 2, k.n_t - 1);
            // staged bins [lo', lo' + TW) with lo' + TW <= n_t - 1 where the
            // row is long enough, so every staged bin has a successor; the
            // window still covers every unit's base bin, with a bin of
            // rounding margin.  A (range-gated) row shorter than TW + 1 bins
            // is staged from bin 0, bins past n_t - 2 clamped below: no unit
            // reads them (its base bin is <= xhi <= n_t - 3).
            const int los = max(0, min(lo, k.n_t - 1 - TW));
            const bool fast = xlo >= 1.f && xhi <= k.xmax - 2.f && hi - lo + 1 <= TW;
            const unsigned off = (unsigned)(t * TW - los) * 16u - LP_MAGIC_BITS * 16u;
            s_el[t] = make_float4(e.x, e.y, e.z, __int_as_float(fast ? (int)off : -1));
            s_lo[t] = fast ? los : -1;
            s_row[t] = (e0 + c0 + t) * (int64_t)k.n_t;
            el_fast = fast;
        }
        // block-uniform: every element of the chunk takes the staged path
        const bool all_fast = __syncthreads_and(el_fast);
#pragma unroll 2
        for (int q = t; q < cn * TW; q += LPT) {
            const int j = q >> lw, lo = s_lo[j];
            if (lo < 0) continue;
            const int bin = min(lo + (q & (TW - 1)), k.n_t - 2);
            const float2 *row = env + (s_row[j] + bin);
            const float2 v0 = __ldg(row), v1 = __ldg(row + 1);
            const float2 r = __ldg(rot + bin);
            const float2 a = cmul(v0, r), b2 = cmul(make_float2(v1.x - v0.x, v1.y - v0.y), r);
            s_env[q] = make_float4(a.x, a.y, b2.x, b2.y);
        }
        __syncthreads();
        // one element against this thread's P points: the fast (staged) unit
        auto fast_unit = [&](const float4 &e) {
            const unsigned base = (unsigned)__float_as_int(e.w);
            const f2x nex = bc2(-e.x), ney = bc2(-e.y), nez = bc2(-e.z);
#pragma unroll
            for (int q = 0; q < P; q += 2) {
                const f2x dx = add2(pk2(px[q], px[q + 1]), nex);
                const f2x dy = add2(pk2(py[q], py[q + 1]), ney);
                const f2x dz = add2(pk2(pz[q], pz[q + 1]), nez);
                const f2x a2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
                const f2x d = pk2(lp_sqrt(lo2(a2)), lp_sqrt(hi2(a2)));
                const f2x tb = add2(fma2(d, bc2(k.inv_bin), bc2(k.cbin)), bc2(LP_MAGIC));
                const f2x f = fma2(d, bc2(k.inv_bin), sub2(bc2(k.kfrac), tb));
                const unsigned i0 = (unsigned)__float_as_int(lo2(tb)) * 16u + base;
                const unsigned i1 = (unsigned)__float_as_int(hi2(tb)) * 16u + base;
                const float4 w0 =
                    *reinterpret_cast<const float4 *>(reinterpret_cast<const char *>(s_env) + i0);
                const float4 w1 =
                    *reinterpret_cast<const float4 *>(reinterpret_cast<const char *>(s_env) + i1);
                const f2x v0 = fma2(bc2(lo2(f)), pk2(w0.z, w0.w), pk2(w0.x, w0.y));
                const f2x v1 = fma2(bc2(hi2(f)), pk2(w1.z, w1.w), pk2(w1.x, w1.y));
                const f2x ang = mul2(f, bc2(k.alpha));
                float s0, cs0, s1, cs1;
                __sincosf(lo2(ang), &s0, &cs0);
                __sincosf(hi2(ang), &s1, &cs1);
                pa[q] = fma2(v0, bc2(cs0), pa[q]);
                pb[q] = fma2(v0, bc2(s0), pb[q]);
                pa[q + 1] = fma2(v1, bc2(cs1), pa[q + 1]);
                pb[q + 1] = fma2(v1, bc2(s1), pb[q + 1]);
            }
        };
        // checked path: exact reference skip-and-count, global gathers
        auto checked_unit = [&](const float4 &e, int j) {
            const float2 *row = env + (e0 + c0 + j) * (int64_t)k.n_t;
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const float dx = px[q] - e.x, dy = py[q] - e.y, dz = pz[q] - e.z;
                const float d = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                const float x = fmaf(d, k.inv_bin, -k.x0);
                if (!(x >= 0.f && x <= k.xmax)) {
                    bad += lat[q] >= 0;
                    continue;
                }
                const int ib = min((int)x, k.n_t - 2);
                const float fr = x - (float)ib;
                const float2 u0 = __ldg(row + ib), u1 = __ldg(row + ib + 1);
                const float er = fmaf(fr, u1.x - u0.x, u0.x), ei = fmaf(fr, u1.y - u0.y, u0.y);
                const float rv = d * k.rev;
                float s, cs;
                __sincosf(6.283185307f * __fsub_rn(rv, rintf(rv)), &s, &cs);
                pa[q] = add2(pa[q], pk2(er * cs - ei * s, er * s + ei * cs));
            }
        };
        // elements two at a time (loop overhead and the element load shared;
        // two independent unit chains in flight)
        int j = warp_live ? 0 : cn;  // warps without points only stage
        if (all_fast) {  // the common case: no per-element path test
            for (; j + 3 < cn; j += 4) {
                const float4 ea = s_el[j], eb = s_el[j + 1], ec = s_el[j + 2], ed = s_el[j + 3];
                fast_unit(ea);
                fast_unit(eb);
                fast_unit(ec);
                fast_unit(ed);
            }
        }
        for (; j + 1 < cn; j += 2) {
            const float4 ea = s_el[j], eb = s_el[j + 1];
            if (__float_as_int(ea.w) != -1 && __float_as_int(eb.w) != -1) {
                fast_unit(ea);
                fast_unit(eb);
            } else {
                if (__float_as_int(ea.w) != -1) fast_unit(ea); else checked_unit(ea, j);
                if (__float_as_int(eb.w) != -1) fast_unit(eb); else checked_unit(eb, j + 1);
            }
        }
        if (j < cn) {
            const float4 e = s_el[j];
            if (__float_as_int(e.w) != -1) fast_unit(e); else checked_unit(e, j);
        }
    }
    const double gap = box_gap_exact(D.ext);
#pragma unroll
    for (int q = 0; q < P; ++q) {
        if (lat[q] < 0) continue;
        float2 v = make_float2(lo2(pa[q]) - hi2(pb[q]), hi2(pa[q]) + lo2(pb[q]));
        if (downconvert) {
            const double *pp = positions + 3 * (D.offset + lat[q]);
            const double phi = sdc_phase_fast(D.ext, gap, g.k_min, g.k_max, pp[0], pp[1], pp[2]);
            v = cmul(v, cis_reduced(-phi));
        }
        values[D.offset + lat[q]] = v;
    }
    if (bad) atomicAdd((unsigned long long *)oow_total, (unsigned long long)bad);
}

int launch_leaf_points(const hhsar_grid_desc *grids, int64_t n_grids, int64_t max_points,
                       int64_t pool_begin, int64_t pool_end, const double *positions,
                       const uint8_t *valid, const float4 *el, const float2 *env, int64_t n_t,
                       double t0, double dt, double k_ref, const hhsar_geom &g, int downconvert,
                       float2 *values, int64_t *oow_total, cudaStream_t s) {
    constexpr int P = 2;  // 512-point chunks: finer fill and 40 registers (P = 4: +8% at config 4)
    LeafFast k;
    k.inv_bin = (float)(2.0 / (HHSAR_C_LIGHT * dt));
    k.x0 = (float)(t0 / dt);
    k.xmax = (float)(n_t - 1);
    k.cbin = -0.5f - k.x0;
    k.kfrac = LP_MAGIC - k.x0;
    k.alpha_d = k_ref * HHSAR_C_LIGHT * dt;
    k.alpha = (float)k.alpha_d;
    k.kc_t0 = k_ref * HHSAR_C_LIGHT * t0;
    k.rev = (float)(k_ref / 3.141592653589793);
    k.n_t = (int)n_t;
    int32_t *idx = nullptr, *cnt = nullptr;
    float2 *rot = nullptr;
    const int64_t pool = pool_end;  // idx is indexed by global lattice offsets
    if (cudaMallocAsync(&idx, pool * sizeof(int32_t), s) != cudaSuccess ||
        cudaMallocAsync(&cnt, n_grids * sizeof(int32_t), s) != cudaSuccess ||
        cudaMallocAsync(&rot, n_t * sizeof(float2), s) != cudaSuccess)
        return set_error(HHSAR_ECUDA, "leaf_bp: scratch allocation failed");
    leaf_rot_kernel<<<(unsigned)((n_t + 255) / 256), 256, 0, s>>>(rot, (int)n_t, k.kc_t0, k.alpha_d);
    // masked lattice points carry 0 (ffbp.py:174-175); valid ones are written below
    cudaMemsetAsync(values + pool_begin, 0, (pool_end - pool_begin) * sizeof(float2), s);
    compact_leaf_kernel<<<(unsigned)n_grids, LP_THREADS, 0, s>>>(grids, valid, idx, cnt);
    const int chunks = (int)((max_points + LPT * P - 1) / (LPT * P));
    const unsigned blocks = (unsigned)(n_grids * chunks);
    leaf_points_kernel<P><<<blocks, LPT, 0, s>>>(
        grids, chunks, idx, cnt, positions, el, env, rot, k, g, downconvert, values, oow_total);
    cudaFreeAsync(idx, s);
    cudaFreeAsync(cnt, s);
    cudaFreeAsync(rot, s);
    return check_launch("leaf_points_kernel");
}

}  // namespace hhsar
