// Level-1 subimages, point-list form (reference: ffbp.py:310-348).
//
// 1. compact_leaf_kernel: per leaf grid, an ordered list of its valid
//    lattice points (block scan; lattice order keeps a CTA's points compact:
//    a few (u, v) columns, n fastest).
// 2. leaf_points_kernel: CTA = (leaf, chunk of 256 x P compacted points).
//    Same unit as the Cartesian BPA tile kernel: per element a delay window
//    of TW bins covering the chunk's bounding box is staged in shared memory
//    pre-rotated by the carrier, points are processed in pairs with packed
//    fp32x2 arithmetic; elements whose window does not fit take a checked
//    global-gather path (reference skip-and-count semantics).  Epilogue:
//    spatial downconversion exp(-j Phi_leaf(pos)) in float64, store to the
//    point's lattice slot (masked slots are zeroed beforehand).
#include "common.cuh"

namespace hhsar {

constexpr int LP_THREADS = 256;
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
    const int npts = D.dims[0] * D.dims[1] * D.dims[2];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int running = 0;
    for (int c0 = 0; c0 < npts; c0 += LP_THREADS) {
        const int i = c0 + threadIdx.x;
        const bool f = i < npts && valid[D.offset + i];
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

__device__ __forceinline__ float lp_sqrt(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

template <int P, int TW>
__global__ void __launch_bounds__(LP_THREADS)
leaf_points_kernel(const hhsar_grid_desc *__restrict__ grids, int chunks,
                   const int32_t *__restrict__ idx, const int32_t *__restrict__ cnt,
                   const double *__restrict__ positions, const float4 *__restrict__ el,
                   const float2 *__restrict__ env, LeafFast k, hhsar_geom g, int downconvert,
                   float2 *__restrict__ values, int64_t *__restrict__ oow_total) {
    static_assert(P % 2 == 0, "points are processed in pairs");
    constexpr int LP_CHUNK = 2048 / TW;  // elements per staging pass: 32 KB of windows
    __shared__ float4 s_env[LP_CHUNK * TW];
    __shared__ float4 s_el[LP_CHUNK];
    __shared__ int s_lo[LP_CHUNK];
    __shared__ float s_box[6][LP_THREADS / 32];
    const int gi = blockIdx.x / chunks, chunk = blockIdx.x % chunks;
    const hhsar_grid_desc &D = grids[gi];
    const int n = cnt[gi];
    const int p0 = chunk * LP_THREADS * P;
    if (p0 >= n) return;  // block-uniform
    const int t = threadIdx.x;
    // my points (strided so a warp's loads are contiguous)
    float px[P], py[P], pz[P];
    int lat[P];
    float mn[3] = {3e38f, 3e38f, 3e38f}, mx[3] = {-3e38f, -3e38f, -3e38f};
#pragma unroll
    for (int q = 0; q < P; ++q) {
        const int li = p0 + q * LP_THREADS + t;
        lat[q] = li < n ? idx[D.offset + li] : -1;
        const int src = lat[q] >= 0 ? lat[q] : idx[D.offset + p0];  // dead lanes mirror a live point
        const double *pp = positions + 3 * (D.offset + src);
        px[q] = (float)pp[0];
        py[q] = (float)pp[1];
        pz[q] = (float)pp[2];
        mn[0] = fminf(mn[0], px[q]);
        mx[0] = fmaxf(mx[0], px[q]);
        mn[1] = fminf(mn[1], py[q]);
        mx[1] = fmaxf(mx[1], py[q]);
        mn[2] = fminf(mn[2], pz[q]);
        mx[2] = fmaxf(mx[2], pz[q]);
    }
    // block bounding box of the chunk's points
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[a] = fminf(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = fmaxf(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
        if ((t & 31) == 0) {
            s_box[a][t >> 5] = mn[a];
            s_box[3 + a][t >> 5] = mx[a];
        }
    }
    __syncthreads();
    float b0[3], b1[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        b0[a] = s_box[a][0];
        b1[a] = s_box[3 + a][0];
        for (int w = 1; w < LP_THREADS / 32; ++w) {
            b0[a] = fminf(b0[a], s_box[a][w]);
            b1[a] = fmaxf(b1[a], s_box[3 + a][w]);
        }
    }
    f2x pa[P], pb[P];
#pragma unroll
    for (int q = 0; q < P; ++q) pa[q] = pb[q] = pk2(0.f, 0.f);
    unsigned bad = 0;
    const int64_t e0 = D.start, m = D.stop - D.start;
    for (int64_t c0 = 0; c0 < m; c0 += LP_CHUNK) {
        const int cn = (int)min((int64_t)LP_CHUNK, m - c0);
        __syncthreads();
        if (t < cn) {
            const float4 e = el[e0 + c0 + t];
            const float qx = fminf(fmaxf(e.x, b0[0]), b1[0]) - e.x;
            const float qy = fminf(fmaxf(e.y, b0[1]), b1[1]) - e.y;
            const float qz = fminf(fmaxf(e.z, b0[2]), b1[2]) - e.z;
            const float fx = fmaxf(fabsf(e.x - b0[0]), fabsf(e.x - b1[0]));
            const float fy = fmaxf(fabsf(e.y - b0[1]), fabsf(e.y - b1[1]));
            const float fz = fmaxf(fabsf(e.z - b0[2]), fabsf(e.z - b1[2]));
            const float xlo = sqrtf(qx * qx + qy * qy + qz * qz) * k.inv_bin - k.x0;
            const float xhi = sqrtf(fx * fx + fy * fy + fz * fz) * k.inv_bin - k.x0;
            const int lo = max((int)floorf(xlo) - 2, 0);
            const int hi = min((int)floorf(xhi) + 2, k.n_t - 1);
            const bool fast = xlo >= 1.f && xhi <= k.xmax - 1.f && hi - lo + 1 <= TW;
            const unsigned off = (unsigned)(t * TW - lo) * 16u - LP_MAGIC_BITS * 16u;
            s_el[t] = make_float4(e.x, e.y, e.z, __int_as_float(fast ? (int)off : -1));
            s_lo[t] = fast ? lo : -1;
        }
        __syncthreads();
        for (int q = t; q < cn * TW; q += LP_THREADS) {
            const int j = q / TW, lo = s_lo[j];
            if (lo < 0) continue;
            const int bin = lo + (q % TW);
            const float2 *row = env + (e0 + c0 + j) * (int64_t)k.n_t;
            const float2 v0 = __ldg(row + min(bin, k.n_t - 1));
            const float2 v1 = __ldg(row + min(bin + 1, k.n_t - 1));
            const float2 r = cis_reduced(k.kc_t0 + k.alpha_d * (double)bin);
            const float2 dv = bin < k.n_t - 1 ? make_float2(v1.x - v0.x, v1.y - v0.y)
                                              : make_float2(0.f, 0.f);
            const float2 a = cmul(v0, r), b2 = cmul(dv, r);
            s_env[q] = make_float4(a.x, a.y, b2.x, b2.y);
        }
        __syncthreads();
        for (int j = 0; j < cn; ++j) {
            const float4 e = s_el[j];
            const int offb = __float_as_int(e.w);
            if (offb != -1) {
                const unsigned base = (unsigned)offb;
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
            } else {
                // checked path: exact reference skip-and-count, global gathers
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
            }
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
    constexpr int P = 4;
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
    const int64_t pool = pool_end;  // idx is indexed by global lattice offsets
    if (cudaMallocAsync(&idx, pool * sizeof(int32_t), s) != cudaSuccess ||
        cudaMallocAsync(&cnt, n_grids * sizeof(int32_t), s) != cudaSuccess)
        return set_error(HHSAR_ECUDA, "leaf_bp: scratch allocation failed");
    // masked lattice points carry 0 (ffbp.py:174-175); valid ones are written below
    cudaMemsetAsync(values + pool_begin, 0, (pool_end - pool_begin) * sizeof(float2), s);
    compact_leaf_kernel<<<(unsigned)n_grids, LP_THREADS, 0, s>>>(grids, valid, idx, cnt);
    const int chunks = (int)((max_points + LP_THREADS * P - 1) / (LP_THREADS * P));
    // window width: a chunk's points span up to the region's depth + lateral
    // extent; in delay bins that is ~ (region diagonal) / (c dt / 2)
    const double rd = sqrt(pow(g.region[1] - g.region[0], 2) + pow(g.region[3] - g.region[2], 2) +
                           pow(g.region[5] - g.region[4], 2));
    const double bins = 1.25 * rd * 2.0 / (HHSAR_C_LIGHT * dt) + 6.0;  // + pad-shell overhang
    const unsigned blocks = (unsigned)(n_grids * chunks);
    if (bins <= 64)
        leaf_points_kernel<P, 64><<<blocks, LP_THREADS, 0, s>>>(
            grids, chunks, idx, cnt, positions, el, env, k, g, downconvert, values, oow_total);
    else if (bins <= 128)
        leaf_points_kernel<P, 128><<<blocks, LP_THREADS, 0, s>>>(
            grids, chunks, idx, cnt, positions, el, env, k, g, downconvert, values, oow_total);
    else
        leaf_points_kernel<P, 256><<<blocks, LP_THREADS, 0, s>>>(
            grids, chunks, idx, cnt, positions, el, env, k, g, downconvert, values, oow_total);
    cudaFreeAsync(idx, s);
    cudaFreeAsync(cnt, s);
    return check_launch("leaf_points_kernel");
}

}  // namespace hhsar
