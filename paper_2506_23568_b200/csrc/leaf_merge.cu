// Level-1 subimages and the merge stages (reference: ffbp.py:310-412 and
// ffbp.py:493-495; interpolation _kernels.py:117-200).
//
// Leaf BPA (hhsar_leaf_bp): the C-ABI entry point; the kernel lives in
// leaf2.cu (leaf_points_kernel: compacted valid points, delay windows staged
// in shared memory, downconversion exp(-j Phi(pos)) (ffbp.py:343-348) fused
// into the store so the lattice is ready for the next level).
//
// Merge: one thread per parent lattice point (or Cartesian voxel).  For every
// child: compressed coordinates (float64), lattice interpolation of the
// child's downconverted complex64 values, and one combined phase
// exp(j (Phi_child(p) - Phi_parent(p))) -- re-modulation by the child and
// downconversion for the next level in a single float64 difference.
#include "common.cuh"

namespace hhsar {

constexpr int MERGE_THREADS = 128;

#ifndef HHSAR_LANDING_TILE
#define HHSAR_LANDING_TILE 16  // landing: a warp's columns (x 32 / TILE z blocks); 0: linear order
#endif

__device__ __forceinline__ int find_by_offset(const hhsar_grid_desc *__restrict__ grids, int n,
                                              int64_t key) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (grids[mid].offset <= key) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ---- merge stages -----------------------------------------------------------
// Per-child constants of one merge launch, prepared once (merge_prep_kernel)
// so the per-point loop reads them instead of re-deriving them (and pays no
// float64 -> float32 conversions on the XU pipe per point and child).
struct __align__(16) MergeChild {
    double ext[4];   // lateral element bbox
    double o_n;      // lattice origin along n
    double gap;      // 4 dx^2 + 4 dy^2 (spectrum.py:142-144)
    int64_t offset;  // first lattice point in the value pool
    int32_t nu, nv, nn, pad_;
    float ef[4];     // ext as float32
    float ku, kv;    // c_uv * width / step (u, v lattice units per unit of the float form)
    float ou, ov;    // -origin_{u,v} / step
    float hu, hv;    // largest interpolation base along u, v (n - 2 linear, n - 3 cubic)
};

__global__ void merge_prep_kernel(const hhsar_grid_desc *__restrict__ d, int n, hhsar_geom g,
                                  int kernel, MergeChild *__restrict__ out,
                                  const hhsar_grid_desc *__restrict__ parents, int n_parents,
                                  int n_blocks, int32_t *__restrict__ block_parent) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) {
        // then the parent of every merge block's first point (the merge
        // kernel walks forward from it instead of a per-point search)
        i -= n;
        if (i < n_blocks)
            block_parent[i] = find_by_offset(parents, n_parents,
                                             parents[0].offset + (int64_t)i * MERGE_THREADS);
        return;
    }
    const hhsar_grid_desc &D = d[i];
    MergeChild c;
    const double inv_step = 1.0 / g.step;
    for (int k = 0; k < 4; ++k) {
        c.ext[k] = D.ext[k];
        c.ef[k] = (float)D.ext[k];
    }
    const double wx = D.ext[1] - D.ext[0], wy = D.ext[3] - D.ext[2];
    c.o_n = D.origin[2];
    c.gap = 4.0 * (wx * wx) + 4.0 * (wy * wy);
    c.offset = D.offset;
    c.nu = D.dims[0];
    c.nv = D.dims[1];
    c.nn = D.dims[2];
    c.pad_ = 0;
    c.ku = (float)(g.c_uv * wx * inv_step);
    c.kv = (float)(g.c_uv * wy * inv_step);
    c.ou = (float)(-D.origin[0] * inv_step);
    c.ov = (float)(-D.origin[1] * inv_step);
    c.hu = (float)(D.dims[0] - (kernel ? 3 : 2));
    c.hv = (float)(D.dims[1] - (kernel ? 3 : 2));
    out[i] = c;
}

// 7 x 16-B loads (the struct is 112 B, 16-B aligned)
__device__ __forceinline__ MergeChild load_child(const MergeChild *p) {
    static_assert(sizeof(MergeChild) == 112, "MergeChild layout");
    MergeChild c;
    const uint4 *src = reinterpret_cast<const uint4 *>(p);
    uint4 *dst = reinterpret_cast<uint4 *>(&c);
#pragma unroll
    for (int k = 0; k < 7; ++k) dst[k] = __ldg(src + k);
    return c;
}

// floor(c) for 0 <= c < 2^22 without F2I/I2F (XU pipe): round-down add of
// 1.5 * 2^23 leaves the integer in the low mantissa bits.  Base clamped to hi.
__device__ __forceinline__ void split_f(float c, float hi, int &i, float &f) {
    const float magic = 12582912.0f;
    float b = __fadd_rd(c, magic) - magic;
    b = fminf(b, hi);
    i = __float_as_int(b + magic) - __float_as_int(magic);
    f = c - b;
}
__device__ __forceinline__ void split_d(double c, int hi, int &i, float &f) {
    const double magic = 6755399441055744.0;  // 1.5 * 2^52
    const double t = __dadd_rd(c, magic);
    i = __double2loint(t);
    f = (float)(c - (t - magic));  // exact floor, no int -> double conversion
    if (i > hi) {  // c at the top edge: base hi, fraction 1
        i = hi;
        f += 1.f;
    }
}

// The lattice gather of one sample at integer bases (iu, iv, iw) and
// fractions (fu, fv, fn) (_kernels.py:117-189): trilinear as nested lerps,
// or Keys cubic over the 4 x 4 x 4 neighbourhood.
template <int KERNEL>
__device__ __forceinline__ float2 gather_child(const float2 *__restrict__ vals, const MergeChild &C,
                                               int iu, int iv, int iw, float fu, float fv, float fn) {
    const int su = C.nv * C.nn;  // lattices hold < 2^31 points (int32 dims product)
    const float2 *base = vals + C.offset;
    float2 acc = make_float2(0.f, 0.f);
    if (KERNEL == 0) {
        // trilinear as nested lerps along n, v, u on (re, im) pairs: one
        // FADD2 + one FFMA2 per lerp, no weight products; row addresses from
        // 32-bit lattice indices (one wide multiply-add each)
        const unsigned i00 = (unsigned)((iu * C.nv + iv) * C.nn + iw);
        const unsigned idx[2][2] = {{i00, i00 + (unsigned)C.nn},
                                    {i00 + (unsigned)su, i00 + (unsigned)(su + C.nn)}};
        f2x r[2][2];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int bb = 0; bb < 2; ++bb) {
                const float2 *row = base + idx[a][bb];
                const float2 v0 = __ldg(row), v1 = __ldg(row + 1);
                const f2x x0 = pk2(v0.x, v0.y);
                r[a][bb] = fma2(bc2(fn), sub2(pk2(v1.x, v1.y), x0), x0);
            }
        const f2x s0 = fma2(bc2(fv), sub2(r[0][1], r[0][0]), r[0][0]);
        const f2x s1 = fma2(bc2(fv), sub2(r[1][1], r[1][0]), r[1][0]);
        const f2x a2 = fma2(bc2(fu), sub2(s1, s0), s0);
        acc = make_float2(lo2(a2), hi2(a2));
    } else {
        float wu[4], wv[4], wn[4];
        keys_weights(fu, wu);
        keys_weights(fv, wv);
        keys_weights(fn, wn);
        const float2 *b = base + (((iu - 1) * C.nv + (iv - 1)) * C.nn + (iw - 1));
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                const float2 *row = b + a * su + bb * C.nn;
                const float w = wu[a] * wv[bb];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float2 v = __ldg(row + c);
                    acc.x = fmaf(v.x, w * wn[c], acc.x);
                    acc.y = fmaf(v.y, w * wn[c], acc.y);
                }
            }
    }
    return acc;
}

// one pair-staged stencil row: base + 16 idx as a single wide multiply-add
__device__ __forceinline__ const float4 *pair_row(const float4 *base, unsigned idx) {
    const float4 *p;
    asm("mad.wide.u32 %0, %1, 16, %2;" : "=l"(p) : "r"(idx), "l"(base));
    return p;
}

// The same gather from the pair-staged copy of the child lattices: entry i
// holds (v[i], v[i + 1] - v[i]) in 16 B, so each lattice row of the stencil
// is one 128-bit load (linear: 4 per sample instead of 8; cubic: 32 instead
// of 64).  ``base`` = the pair copy + the child's pool offset, formed once
// per child by the caller; each row address is then pair_row (left to
// itself the compiler re-derives the 64-bit (offset + index) * 16 + pairs
// in four instructions per row).
template <int KERNEL>
__device__ __forceinline__ float2 gather_child_pairs(const float4 *__restrict__ base,
                                                     const MergeChild &C, int iu, int iv, int iw,
                                                     float fu, float fv, float fn) {
    const int su = C.nv * C.nn;
    if (KERNEL == 0) {
        const unsigned i00 = (unsigned)((iu * C.nv + iv) * C.nn + iw);
        const unsigned idx[2][2] = {{i00, i00 + (unsigned)C.nn},
                                    {i00 + (unsigned)su, i00 + (unsigned)(su + C.nn)}};
        f2x r[2][2];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int bb = 0; bb < 2; ++bb) {
                const float4 v = __ldg(pair_row(base, idx[a][bb]));  // (v[i], v[i+1] - v[i])
                r[a][bb] = fma2(bc2(fn), pk2(v.z, v.w), pk2(v.x, v.y));
            }
        const f2x s0 = fma2(bc2(fv), sub2(r[0][1], r[0][0]), r[0][0]);
        const f2x s1 = fma2(bc2(fv), sub2(r[1][1], r[1][0]), r[1][0]);
        const f2x a2 = fma2(bc2(fu), sub2(s1, s0), s0);
        return make_float2(lo2(a2), hi2(a2));
    } else {
        float wu[4], wv[4], wn[4];
        keys_weights(fu, wu);
        keys_weights(fv, wv);
        keys_weights(fn, wn);
        const float4 *b = base + (((iu - 1) * C.nv + (iv - 1)) * C.nn + (iw - 1));
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                const float4 *row = b + a * su + bb * C.nn;
                const float w = wu[a] * wv[bb];
                float4 p0 = __ldg(row), p1 = __ldg(row + 2);  // (v[i], v[i+1] - v[i]) pairs
                p0.z += p0.x;
                p0.w += p0.y;
                p1.z += p1.x;
                p1.w += p1.y;
                acc.x = fmaf(p0.x, w * wn[0], fmaf(p0.z, w * wn[1], fmaf(p1.x, w * wn[2], fmaf(p1.z, w * wn[3], acc.x))));
                acc.y = fmaf(p0.y, w * wn[0], fmaf(p0.w, w * wn[1], fmaf(p1.y, w * wn[2], fmaf(p1.w, w * wn[3], acc.y))));
            }
        return acc;
    }
}

// pairs[i - begin] = (v[i], v[i + 1] - v[i]) for the child lattices' pool
// span: the n-lerp of a stencil row is then one packed FMA
__global__ void pair_rows_kernel(const float2 *__restrict__ vals, int64_t begin, int64_t n,
                                 float4 *__restrict__ pairs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float2 a = vals[begin + i], b = vals[begin + (i + 1 < n ? i + 1 : i)];
    pairs[i] = make_float4(a.x, a.y, b.x - a.x, b.y - a.y);
}

// Lattice interpolation with the reference's hull rules (_kernels.py:117-189)
// on float u, v and double n lattice coordinates.
template <int KERNEL>
__device__ __forceinline__ bool sample_child(const float2 *__restrict__ vals, const MergeChild &C,
                                             float cu, float cv, double cn, float2 &out) {
    out = make_float2(0.f, 0.f);
    const int lo = KERNEL ? 1 : 0;
    if (!(cu >= (float)lo && cu <= C.hu + 1.f && cv >= (float)lo && cv <= C.hv + 1.f &&
          cn >= (double)lo && cn <= (double)(C.nn - 1 - lo)))
        return false;
    int iu, iv, iw;
    float fu, fv, fn;
    split_f(cu, C.hu, iu, fu);
    split_f(cv, C.hv, iv, fv);
    split_d(cn, C.nn - (KERNEL ? 3 : 2), iw, fn);
    out = gather_child<KERNEL>(vals, C, iu, iv, iw, fu, fv, fn);
    return true;
}

__device__ __forceinline__ float sqrt_fast(float a) { return sqrt_approx(a); }

// exp(j phi), float64 phase of any size: reduction by 2 pi with a magic-number
// round (no FRND), then the fp32 SFU sincos.
__device__ __forceinline__ float2 cis_fast(double phi) {
    const double magic = 6755399441055744.0;
    const double n = fma(phi, 0.15915494309189535, magic) - magic;
    float s, c;
    __sincosf((float)fma(-6.283185307179586, n, phi), &s, &c);
    return make_float2(c, s);
}

// Sum over children of interp_child(llt_child(p)) exp(j (Phi_child(p) -
// phi_parent)) at point p (ffbp.py:378-412).  Mixed precision, by what each
// quantity feeds:
// * u, v in float32 via d_a - d_b = (e1 - e0)(a_x + b_x) / (d_a + d_b): no
//   cancellation; absolute error ~1e-7 m in (a_x + b_x), i.e. < 1e-5 lattice
//   steps;
// * the four corner distances, r, sqrt(r^2 - gap), n and the phase in float64
//   (SFU-seeded rsqrt + one Newton step, 1e-13): the phase is ~1e3 rad and a
//   float32 distance would cost ~1e-4 rad per level;
// * lattice coordinates by multiplication with 1/step, floors by magic-number
//   adds (no float64 division, no F2I/I2F).
template <int KERNEL>
__device__ __forceinline__ bool merge_point(const MergeChild *__restrict__ kids, int nk,
                                            const float2 *__restrict__ kv, const hhsar_geom &g,
                                            double inv_step, double x, double y, double z,
                                            double phi_parent, float2 &acc) {
    acc = make_float2(0.f, 0.f);
    bool good = true;
    const float xf = (float)x, yf = (float)y;
    const double z2 = z * z;
    const float z2f = (float)z2;
    for (int c = 0; c < nk; ++c) {
        const MergeChild C = load_child(kids + c);
        const float axf = xf - C.ef[0], bxf = xf - C.ef[1], ayf = yf - C.ef[2], byf = yf - C.ef[3];
        const float dx0 = axf < 0.f ? axf : (bxf > 0.f ? bxf : 0.f);  // x - clip(x, e0, e1)
        const float dy0 = ayf < 0.f ? ayf : (byf > 0.f ? byf : 0.f);
        const float dyz = fmaf(dy0, dy0, z2f), dxz = fmaf(dx0, dx0, z2f);
        const float da = sqrt_fast(fmaf(axf, axf, dyz)), db = sqrt_fast(fmaf(bxf, bxf, dyz));
        const float dc = sqrt_fast(fmaf(ayf, ayf, dxz)), dd = sqrt_fast(fmaf(byf, byf, dxz));
        const float cu = fmaf(C.ku * (axf + bxf), rcp_approx(da + db), C.ou);
        const float cv = fmaf(C.kv * (ayf + byf), rcp_approx(dc + dd), C.ov);
        const double ax = x - C.ext[0], bx = x - C.ext[1], ay = y - C.ext[2], by = y - C.ext[3];
        const double xa = ax * ax, xb = bx * bx, ya = ay * ay, yb = by * by;
        const double r = ((sqrt_d(xa + ya + z2) + sqrt_d(xa + yb + z2)) + sqrt_d(xb + ya + z2)) +
                         sqrt_d(xb + yb + z2);
        const double sq = sqrt_d(fma(r, r, -C.gap));
        const double cn = (fma(g.c_nhi, sq, -g.c_nlo * r) - C.o_n) * inv_step;
        float2 s;
        const bool ok = sample_child<KERNEL>(kv, C, cu, cv, cn, s);
        good &= ok;
        if (ok) cfma(acc, s, cis_fast(fma(0.25 * g.k_max, sq, 0.25 * g.k_min * r) - phi_parent));
    }
    if (!good) acc = make_float2(0.f, 0.f);
    return good;
}

template <int KERNEL>
__global__ void __launch_bounds__(MERGE_THREADS, KERNEL ? 8 : 12)
merge_level_kernel(const hhsar_grid_desc *__restrict__ parents, int n_parents, int64_t n_points,
                   const double *__restrict__ positions, const uint8_t *__restrict__ valid,
                   const MergeChild *__restrict__ kids, int fanout,
                   const float2 *__restrict__ kv, hhsar_geom g, int downconvert,
                   float2 *__restrict__ out, int64_t *__restrict__ flagged,
                   const int32_t *__restrict__ block_parent) {
    const int64_t base = parents[0].offset;
    const int64_t i = base + (int64_t)blockIdx.x * MERGE_THREADS + threadIdx.x;
    if (i >= base + n_points) return;
    // independent loads first: flag, position, the block's first parent
    const uint8_t vi = valid[i];
    const double x = positions[3 * i], y = positions[3 * i + 1], z = positions[3 * i + 2];
    int p = block_parent[blockIdx.x];
    unsigned fl = 0;
    if (vi) {
        while (p + 1 < n_parents && parents[p + 1].offset <= i) ++p;
        const hhsar_grid_desc &P = parents[p];
        const double phi_p =
            downconvert ? sdc_phase_fast(P.ext, box_gap_exact(P.ext), g.k_min, g.k_max, x, y, z)
                        : 0.0;
        float2 acc;
        fl = !merge_point<KERNEL>(kids + (int64_t)p * fanout, fanout, kv, g, rcp_d(g.step), x, y,
                                  z, phi_p, acc);
        out[i] = acc;
    } else {
        out[i] = make_float2(0.f, 0.f);
    }
    warp_add(flagged, fl);
}

// Cartesian landing, ZQ consecutive z voxels of one (x, y) column per
// thread: the child constants and every x/y-only term (lateral offsets,
// their squares, the clamped u/v offsets) are computed once for the ZQ
// voxels; the per-voxel work is the same merge_point arithmetic.  ZQ = 4 or
// 2, chosen at launch (hhsar_merge_cartesian).
template <int KERNEL, int ZQ, int NK = 0>
__global__ void __launch_bounds__(MERGE_THREADS)
merge_cartesian_kernel(double ox, double oy, double oz, double sx, double sy, double sz, int nx,
                       int ny, int nz, int64_t vb, int64_t ve, int64_t q0, int64_t nq,
                       const MergeChild *__restrict__ kids, int nk,
                       const float2 *__restrict__ kv, hhsar_geom g, float2 *__restrict__ out,
                       int64_t *__restrict__ flagged) {
    const int64_t qi = (int64_t)blockIdx.x * MERGE_THREADS + threadIdx.x;
    if (qi >= nq) return;
    const int nzq = (nz + ZQ - 1) / ZQ;
    const int64_t Q = q0 + qi;           // global quad: row (ix, iy), z block k
    const int64_t row = Q / nzq;
    const int k = (int)(Q - row * nzq);
    const int iy = (int)(row % ny), ix = (int)(row / ny);
    (void)nx;
    const double x = __dadd_rn(ox, __dmul_rn(sx, (double)ix));
    const double y = __dadd_rn(oy, __dmul_rn(sy, (double)iy));
    const float xf = (float)x, yf = (float)y;
    const double inv_step = rcp_d(g.step);
    double z[ZQ], z2[ZQ];
    float z2f[ZQ];
    bool live[ZQ];
    float2 acc[ZQ];
    bool good[ZQ];
#pragma unroll
    for (int j = 0; j < ZQ; ++j) {
        const int iz = k * ZQ + j;
        const int64_t v = row * nz + iz;
        live[j] = iz < nz && v >= vb && v < ve;
        z[j] = __dadd_rn(oz, __dmul_rn(sz, (double)iz));
        z2[j] = z[j] * z[j];
        z2f[j] = (float)z2[j];
        acc[j] = make_float2(0.f, 0.f);
        good[j] = true;
    }
    constexpr int UNROLL = NK > 0 ? NK : 1;
#pragma unroll UNROLL
    for (int c = 0; c < (NK > 0 ? NK : nk); ++c) {
        const MergeChild C = load_child(kids + c);
        const float axf = xf - C.ef[0], bxf = xf - C.ef[1], ayf = yf - C.ef[2], byf = yf - C.ef[3];
        const float dx0 = axf < 0.f ? axf : (bxf > 0.f ? bxf : 0.f);  // x - clip(x, e0, e1)
        const float dy0 = ayf < 0.f ? ayf : (byf > 0.f ? byf : 0.f);
        const float nu_ = C.ku * (axf + bxf), nv_ = C.kv * (ayf + byf);
        const float ax2 = axf * axf, bx2 = bxf * bxf, ay2 = ayf * ayf, by2 = byf * byf;
        const float dy02 = dy0 * dy0, dx02 = dx0 * dx0;
        const double ax = x - C.ext[0], bx = x - C.ext[1], ay = y - C.ext[2], by = y - C.ext[3];
        const double s_aa = fma(ax, ax, ay * ay), s_ab = fma(ax, ax, by * by);
        const double s_ba = fma(bx, bx, ay * ay), s_bb = fma(bx, bx, by * by);
#pragma unroll
        for (int j = 0; j < ZQ; ++j) {
            const float dyz = dy02 + z2f[j], dxz = dx02 + z2f[j];
            const float da = sqrt_fast(ax2 + dyz), db = sqrt_fast(bx2 + dyz);
            const float dc = sqrt_fast(ay2 + dxz), dd = sqrt_fast(by2 + dxz);
            const float cu = fmaf(nu_, rcp_approx(da + db), C.ou);
            const float cv = fmaf(nv_, rcp_approx(dc + dd), C.ov);
            const double r = ((sqrt_d(s_aa + z2[j]) + sqrt_d(s_ab + z2[j])) + sqrt_d(s_ba + z2[j])) +
                             sqrt_d(s_bb + z2[j]);
            const double sq = sqrt_d(fma(r, r, -C.gap));
            const double cn = (fma(g.c_nhi, sq, -g.c_nlo * r) - C.o_n) * inv_step;
            float2 smp;
            const bool ok = sample_child<KERNEL>(kv, C, cu, cv, cn, smp);
            good[j] &= ok;
            if (ok) cfma(acc[j], smp, cis_fast(fma(0.25 * g.k_max, sq, 0.25 * g.k_min * r)));
        }
    }
    unsigned fl = 0;
#pragma unroll
    for (int j = 0; j < ZQ; ++j) {
        if (!live[j]) continue;
        fl += !good[j];
        out[row * nz + k * ZQ + j - vb] = good[j] ? acc[j] : make_float2(0.f, 0.f);
    }
    warp_add(flagged, fl);
}

// Cartesian landing along z by Taylor series.  Per (column, child) the
// quantities a voxel needs -- the u and v lattice coordinates, the n
// coordinate and the phase 0.25 (k_max sq + k_min r) -- are smooth in z, so
// a thread owning ZQ consecutive z voxels evaluates them once, with their
// first four z-derivatives, at the block's centre z_c and then per voxel as
// quartic polynomials in t = (z - z_c) / sz (|t| <= (ZQ - 1) / 2):
// * r = sum of the four corner distances d_i = sqrt(s_i + z^2):
//   d_i^(k)/k! from y_i = 1/d_i (float64: s_i y_i^3 / 2, -s_i z y_i^5 / 2,
//   s_i (4 z^2 - s_i) y_i^7 / 8); sq = sqrt(r^2 - gap) by the series square
//   root of r^2 - gap; n and the phase are linear in (r, sq);
// * u = c_uv w_x (a_x + b_x) / (d_a + d_b) by the series reciprocal of the
//   clamped-lateral distance sum (float32, as the per-voxel form).
// Per voxel the n coordinate is an integer base per block plus a float32
// polynomial, and the phase's float32 polynomial starts from the block's
// float64-reduced phase, so no float64 and no square root or reciprocal
// remain per voxel (the per-voxel form: five float64 square roots, four
// fp32 square roots, two reciprocals).  Truncation (fifth order) is
// (ZQ sz / 2d)^5-small: <= 3e-7 rad of phase at config 3 (ZQ = 8, d >= 0.2
// m), 7e-11 at config 4; the launcher falls back to the per-voxel kernel
// when the region's nearest z is not far enough from the aperture plane.
template <int KERNEL, int ZQ>
__global__ void __launch_bounds__(MERGE_THREADS)
merge_cartesian_series_kernel(double ox, double oy, double oz, double sx, double sy, double sz,
                              int ny, int nz, int64_t vb, int64_t ve, int64_t q0, int64_t nq,
                              const MergeChild *__restrict__ kids, int nk,
                              const float2 *__restrict__ kv, const float4 *__restrict__ kp,
                              hhsar_geom g, float2 *__restrict__ out,
                              int64_t *__restrict__ flagged, int tile) {
    int64_t row;  // column (ix, iy) = ix * ny + iy
    int k, ix, iy;  // z block, column
    if (tile) {
        // whole volume, 3-D grid (ny / TC, nzq / (4 TK), nx): a warp takes
        // TC adjacent columns x TK = 32 / TC adjacent z blocks (16 x 2) --
        // its lanes' taps share lattice rows and lines -- and a CTA's four
        // warps take adjacent z-block tiles; no integer division anywhere
        constexpr int TC = HHSAR_LANDING_TILE > 0 ? HHSAR_LANDING_TILE : 1, TK = 32 / TC;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        ix = blockIdx.z;
        iy = blockIdx.x * TC + lane / TK;
        k = (blockIdx.y * (MERGE_THREADS / 32) + warp) * TK + lane % TK;
        row = (int64_t)ix * ny + iy;
    } else {
        const int64_t qi = (int64_t)blockIdx.x * MERGE_THREADS + threadIdx.x;
        if (qi >= nq) return;
        const int nzq = (nz + ZQ - 1) / ZQ;
        const int64_t Q = q0 + qi;
        row = Q / nzq;
        k = (int)(Q - row * nzq);
        iy = (int)(row % ny);
        ix = (int)(row / ny);
    }
    const double x = __dadd_rn(ox, __dmul_rn(sx, (double)ix));
    const double y = __dadd_rn(oy, __dmul_rn(sy, (double)iy));
    const float xf = (float)x, yf = (float)y;
    const double inv_step = rcp_d(g.step);
    const double zc = oz + sz * ((double)(k * ZQ) + 0.5 * (ZQ - 1));
    const double zc2 = zc * zc;
    const float zcf = (float)zc, zc2f = (float)zc2;
    const double sz2 = sz * sz, sz3 = sz2 * sz, sz4 = sz2 * sz2;
    const float szf = (float)sz, sz2f = szf * szf, sz3f = sz2f * szf, sz4f = sz2f * sz2f;
    float2 acc[ZQ];
    unsigned good = (1u << ZQ) - 1u;
#pragma unroll
    for (int j = 0; j < ZQ; ++j) acc[j] = make_float2(0.f, 0.f);
    constexpr int lo = KERNEL ? 1 : 0;
    for (int c = 0; c < nk; ++c) {
        const MergeChild C = load_child(kids + c);
        const float4 *kpc = kp ? kp + C.offset : nullptr;  // this child's pair rows
        // ---- n coordinate and phase: float64 series of r and sq at z_c
        const double ax = x - C.ext[0], bx = x - C.ext[1], ay = y - C.ext[2], by = y - C.ext[3];
        const double ss[4] = {fma(ax, ax, ay * ay), fma(ax, ax, by * by), fma(bx, bx, ay * ay),
                              fma(bx, bx, by * by)};
        double R0 = 0.0, R1 = 0.0, R2 = 0.0, R3 = 0.0, R4 = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double a = ss[i] + zc2, yi = rsqrt_d(a);
            const double y2 = yi * yi, y3 = y2 * yi, y5 = y3 * y2, y7 = y5 * y2;
            R0 += a * yi;
            R1 += yi;
            R2 += ss[i] * y3;
            R3 += ss[i] * y5;
            R4 += ss[i] * fma(4.0, zc2, -ss[i]) * y7;
        }
        R1 *= zc;
        R2 *= 0.5;
        R3 *= -0.5 * zc;
        R4 *= 0.125;
        const double U0 = fma(R0, R0, -C.gap), U1 = 2.0 * R0 * R1, U2 = fma(R1, R1, 2.0 * R0 * R2);
        const double U3 = 2.0 * fma(R0, R3, R1 * R2), U4 = fma(2.0 * R0, R4, fma(2.0 * R1, R3, R2 * R2));
        const double w = rsqrt_d(U0), hw = 0.5 * w;
        const double S0 = U0 * w, S1 = U1 * hw, S2 = fma(-S1, S1, U2) * hw;
        const double S3 = fma(-2.0 * S1, S2, U3) * hw, S4 = (U4 - 2.0 * S1 * S3 - S2 * S2) * hw;
        const double cn0 = (fma(g.c_nhi, S0, -g.c_nlo * R0) - C.o_n) * inv_step;
        const double fl0 = floor(cn0);  // clamped to +-2^20 (comparisons: cheaper than fmin/fmax)
        const double I0d = fl0 > -1048576.0 ? (fl0 < 1048576.0 ? fl0 : 1048576.0) : -1048576.0;
        const int I0 = (int)I0d;
        const float f0 = (float)(cn0 - I0d);
        const float n1 = (float)(fma(g.c_nhi, S1, -g.c_nlo * R1) * inv_step * sz);
        const float n2 = (float)(fma(g.c_nhi, S2, -g.c_nlo * R2) * inv_step * sz2);
        const float n3 = (float)(fma(g.c_nhi, S3, -g.c_nlo * R3) * inv_step * sz3);
        const float n4 = (float)(fma(g.c_nhi, S4, -g.c_nlo * R4) * inv_step * sz4);
        const float n_lo = (float)(lo - I0), n_hi = (float)(C.nn - 1 - lo - I0);
        const float n_base_hi = (float)(C.nn - (KERNEL ? 3 : 2) - I0);
        const double ph0 = 0.25 * fma(g.k_max, S0, g.k_min * R0);
        const float p0 = (float)fma(-6.283185307179586, rint(ph0 * 0.15915494309189535), ph0);
        const float p1 = (float)(0.25 * fma(g.k_max, S1, g.k_min * R1) * sz);
        const float p2 = (float)(0.25 * fma(g.k_max, S2, g.k_min * R2) * sz2);
        const float p3 = (float)(0.25 * fma(g.k_max, S3, g.k_min * R3) * sz3);
        const float p4 = (float)(0.25 * fma(g.k_max, S4, g.k_min * R4) * sz4);
        // ---- u, v coordinates: float32 series of 1 / (d_a + d_b)
        const float axf = xf - C.ef[0], bxf = xf - C.ef[1], ayf = yf - C.ef[2], byf = yf - C.ef[3];
        const float dx0 = axf < 0.f ? axf : (bxf > 0.f ? bxf : 0.f);  // x - clip(x, e0, e1)
        const float dy0 = ayf < 0.f ? ayf : (byf > 0.f ? byf : 0.f);
        float cu_k[5], cv_k[5];
        {
            const float qs[4] = {fmaf(axf, axf, dy0 * dy0), fmaf(bxf, bxf, dy0 * dy0),
                                 fmaf(ayf, ayf, dx0 * dx0), fmaf(byf, byf, dx0 * dx0)};
            float D[2][5];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int m = 0; m < 5; ++m) D[h][m] = 0.f;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float a = qs[i] + zc2f, yi = rsqrt_approx(a);
                const float y2 = yi * yi, y3 = y2 * yi, y5 = y3 * y2, y7 = y5 * y2;
                float *Dh = D[i >> 1];
                Dh[0] += a * yi;
                Dh[1] += zcf * yi;
                Dh[2] += 0.5f * qs[i] * y3;
                Dh[3] += -0.5f * qs[i] * zcf * y5;
                Dh[4] += 0.125f * qs[i] * fmaf(4.f, zc2f, -qs[i]) * y7;
            }
            const float num[2] = {C.ku * (axf + bxf), C.kv * (ayf + byf)};
            const float off[2] = {C.ou, C.ov};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float Cr[5];
                const float inv = rcp_approx(D[h][0]);
                Cr[0] = inv;
#pragma unroll
                for (int m = 1; m < 5; ++m) {
                    float acc_m = 0.f;
#pragma unroll
                    for (int q = 1; q <= m; ++q) acc_m = fmaf(D[h][q], Cr[m - q], acc_m);
                    Cr[m] = -acc_m * inv;
                }
                float *o = h ? cv_k : cu_k;
                o[0] = fmaf(num[h], Cr[0], off[h]);
                o[1] = num[h] * Cr[1] * szf;
                o[2] = num[h] * Cr[2] * sz2f;
                o[3] = num[h] * Cr[3] * sz3f;
                o[4] = num[h] * Cr[4] * sz4f;
            }
        }
        // ---- the block's voxels: (u, v) and (n, phase) as packed pairs
        f2x uv_k[5], np_k[5];
        uv_k[0] = pk2(cu_k[0], cv_k[0]);
        np_k[0] = pk2(f0, p0);
        uv_k[1] = pk2(cu_k[1], cv_k[1]);
        np_k[1] = pk2(n1, p1);
        uv_k[2] = pk2(cu_k[2], cv_k[2]);
        np_k[2] = pk2(n2, p2);
        uv_k[3] = pk2(cu_k[3], cv_k[3]);
        np_k[3] = pk2(n3, p3);
        uv_k[4] = pk2(cu_k[4], cv_k[4]);
        np_k[4] = pk2(n4, p4);
        const f2x magic2 = bc2(12582912.0f);
#pragma unroll
        for (int j = 0; j < ZQ; ++j) {
            const f2x tt = bc2((float)j - 0.5f * (float)(ZQ - 1));
            const f2x uv = fma2(tt, fma2(tt, fma2(tt, fma2(tt, uv_k[4], uv_k[3]), uv_k[2]), uv_k[1]),
                                uv_k[0]);
            const f2x np = fma2(tt, fma2(tt, fma2(tt, fma2(tt, np_k[4], np_k[3]), np_k[2]), np_k[1]),
                                np_k[0]);
            const float cu = lo2(uv), cv = hi2(uv), cf = lo2(np), ph = hi2(np);
            if (!(cu >= (float)lo && cu <= C.hu + 1.f && cv >= (float)lo && cv <= C.hv + 1.f &&
                  cf >= n_lo && cf <= n_hi)) {
                good &= ~(1u << j);
                continue;
            }
            // floors of (u, v) by one round-down packed add (as split_f), the
            // bases clamped to (hu, hv) (top edge: fraction 1)
            const f2x fl2 = sub2(add2_rm(uv, magic2), magic2);
            const f2x b2 = pk2(fminf(lo2(fl2), C.hu), fminf(hi2(fl2), C.hv));
            const f2x bm = add2(b2, magic2);
            const int iu = __float_as_int(lo2(bm)) - __float_as_int(12582912.0f);
            const int iv = __float_as_int(hi2(bm)) - __float_as_int(12582912.0f);
            const f2x fuv = sub2(uv, b2);
            const float fu = lo2(fuv), fv = hi2(fuv);
            float bn = __fadd_rd(cf, 12582912.0f) - 12582912.0f;  // floor(cf)
            bn = fminf(bn, n_base_hi);                              // top edge: base hi, fraction 1
            const int iw = I0 + (int)bn;
            const float fn = cf - bn;
            const float2 smp = kp ? gather_child_pairs<KERNEL>(kpc, C, iu, iv, iw, fu, fv, fn)
                                  : gather_child<KERNEL>(kv, C, iu, iv, iw, fu, fv, fn);
#ifdef HHSAR_LANDING_REDUCE
            const float nr = fmaf(ph, 0.15915494f, 12582912.0f) - 12582912.0f;
            const float red = fmaf(nr, 1.7484555e-7f, fmaf(nr, -6.28318548f, ph));
#else
            // |ph| <= pi + |phase change over half a block| (a few to ~20
            // rad): the SFU's own reduction (x / 2 pi rounded once) costs
            // <= |ph| 2^-24 ~ 1e-6 rad here
            const float red = ph;
#endif
            float sn, cs;
            __sincosf(red, &sn, &cs);
            cfma(acc[j], smp, make_float2(cs, sn));
        }
    }
    const int64_t v0 = row * nz + k * ZQ;
    unsigned fl;
    if (k * ZQ + ZQ <= nz && v0 >= vb && v0 + ZQ <= ve) {  // the whole block is in range
        fl = ZQ - __popc(good);
#pragma unroll
        for (int j = 0; j < ZQ; ++j)
            out[v0 + j - vb] = ((good >> j) & 1u) ? acc[j] : make_float2(0.f, 0.f);
    } else {
        fl = 0;
#pragma unroll
        for (int j = 0; j < ZQ; ++j) {
            const int64_t v = v0 + j;
            if (!(k * ZQ + j < nz && v >= vb && v < ve)) continue;
            const bool ok = (good >> j) & 1u;
            fl += !ok;
            out[v - vb] = ok ? acc[j] : make_float2(0.f, 0.f);
        }
    }
    warp_add(flagged, fl);
}

// Per-child constants for a merge launch (stream-ordered scratch).
static int prep_children(const hhsar_grid_desc *kids, int64_t n, const hhsar_geom &g, int kernel,
                         MergeChild **out, cudaStream_t s,
                         const hhsar_grid_desc *parents = nullptr, int n_parents = 0,
                         int n_blocks = 0, int32_t **block_parent = nullptr) {
    // one scratch block: the child records, then (merge levels) the table
    if (cudaMallocAsync(out, n * sizeof(MergeChild) + (size_t)n_blocks * sizeof(int32_t), s) !=
        cudaSuccess)
        return set_error(HHSAR_ECUDA, "merge: scratch allocation failed");
    int32_t *bp = reinterpret_cast<int32_t *>(*out + n);
    if (block_parent) *block_parent = bp;
    const int64_t work = n + n_blocks;
    merge_prep_kernel<<<(unsigned)((work + 127) / 128), 128, 0, s>>>(
        kids, (int)n, g, kernel, *out, parents, n_parents, n_blocks, bp);
    return check_launch("merge_prep_kernel");
}

template <int KERNEL>
__global__ void lattice_interp_kernel(const float2 *__restrict__ vals, int nu, int nv, int nn,
                                      const double *__restrict__ coords, int64_t n,
                                      float2 *__restrict__ out, uint8_t *__restrict__ ok) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float2 s;
    ok[i] = lattice_sample<KERNEL>(vals, nu, nv, nn, coords[3 * i], coords[3 * i + 1],
                                   coords[3 * i + 2], s);
    out[i] = s;
}

// values[i] *= exp(-j Phi_grid(pos_i)) for valid points, 0 elsewhere
// (_downconvert_samples, ffbp.py:343-348) -- used by the single-merge API.
__global__ void downconvert_kernel(const hhsar_grid_desc *__restrict__ grids, int n_grids,
                                   int64_t n_points, const double *__restrict__ positions,
                                   const uint8_t *__restrict__ valid, hhsar_geom g,
                                   float2 *__restrict__ values) {
    const int64_t base = grids[0].offset;
    const int64_t i = base + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= base + n_points) return;
    if (!valid[i]) {
        values[i] = make_float2(0.f, 0.f);
        return;
    }
    const hhsar_grid_desc &D = grids[find_by_offset(grids, n_grids, i)];
    const double phi = sdc_phase_fast(D.ext, box_gap_exact(D.ext), g.k_min, g.k_max,
                                      positions[3 * i], positions[3 * i + 1], positions[3 * i + 2]);
    values[i] = cmul(values[i], cis_reduced(-phi));
}

}  // namespace hhsar

using namespace hhsar;

extern "C" int hhsar_leaf_bp(const hhsar_grid_desc *grids, int64_t n_grids, int64_t point_begin,
                             int64_t point_end, int64_t max_grid_points, const double *positions,
                             const uint8_t *valid, const float *el_xyz, const void *envelopes,
                             int64_t n_t, double t0, double dt, double k_ref,
                             const hhsar_geom *geom, int downconvert, void *values,
                             int64_t *oow_total, void *stream) {
    HHSAR_REQUIRE(n_grids > 0 && n_grids < (1 << 24) && geom, "leaf_bp: bad grid count");
    HHSAR_REQUIRE(n_t >= 2, "leaf_bp: n_t must be >= 2");
    HHSAR_REQUIRE(point_begin >= 0 && point_end >= point_begin && point_end < (1ll << 31) &&
                  max_grid_points >= 0, "leaf_bp: bad point range");
    return launch_leaf_points(grids, n_grids, max_grid_points, point_begin, point_end, positions,
                              valid, reinterpret_cast<const float4 *>(el_xyz),
                              reinterpret_cast<const float2 *>(envelopes), n_t, t0, dt, k_ref,
                              *geom, downconvert, reinterpret_cast<float2 *>(values), oow_total,
                              as_stream(stream));
}

extern "C" int hhsar_merge_level(const hhsar_grid_desc *parent_grids, int64_t n_parents,
                                 int64_t n_parent_points, const double *positions,
                                 const uint8_t *valid, const hhsar_grid_desc *child_grids,
                                 int64_t n_child_grids, int fanout, const void *values_in,
                                 const hhsar_geom *geom, int kernel, int downconvert,
                                 void *values_out, int64_t *flagged, void *stream) {
    HHSAR_REQUIRE(n_parents > 0 && fanout >= 1 && n_child_grids == n_parents * fanout && geom,
                  "merge_level: children must be n_parents * fanout");
    HHSAR_REQUIRE(kernel == 0 || kernel == 1, "merge_level: unknown interpolation kernel");
    if (n_parent_points == 0) return HHSAR_OK;
    const unsigned blocks = (unsigned)((n_parent_points + MERGE_THREADS - 1) / MERGE_THREADS);
    cudaStream_t s = as_stream(stream);
    auto kv = reinterpret_cast<const float2 *>(values_in);
    auto out = reinterpret_cast<float2 *>(values_out);
    MergeChild *kids = nullptr;
    int32_t *block_parent = nullptr;
    int rc = prep_children(child_grids, n_child_grids, *geom, kernel, &kids, s, parent_grids,
                           (int)n_parents, (int)blocks, &block_parent);
    if (rc != HHSAR_OK) return rc;
    if (kernel == 0)
        merge_level_kernel<0><<<blocks, MERGE_THREADS, 0, s>>>(
            parent_grids, (int)n_parents, n_parent_points, positions, valid, kids, fanout,
            kv, *geom, downconvert, out, flagged, block_parent);
    else
        merge_level_kernel<1><<<blocks, MERGE_THREADS, 0, s>>>(
            parent_grids, (int)n_parents, n_parent_points, positions, valid, kids, fanout,
            kv, *geom, downconvert, out, flagged, block_parent);
    rc = check_launch("merge_level_kernel");
    cudaFreeAsync(kids, s);
    return rc;
}

extern "C" int hhsar_downconvert(const hhsar_grid_desc *grids, int64_t n_grids, int64_t n_points,
                                 const double *positions, const uint8_t *valid,
                                 const hhsar_geom *geom, void *values, void *stream) {
    HHSAR_REQUIRE(n_grids > 0 && geom, "downconvert: bad arguments");
    if (n_points == 0) return HHSAR_OK;
    downconvert_kernel<<<(unsigned)((n_points + 255) / 256), 256, 0, as_stream(stream)>>>(
        grids, (int)n_grids, n_points, positions, valid, *geom, reinterpret_cast<float2 *>(values));
    return check_launch("downconvert_kernel");
}
extern "C" int hhsar_merge_cartesian(const double *origin, const double *step, const int64_t *dims,
                                     int64_t vox_begin, int64_t vox_end,
                                     const hhsar_grid_desc *child_grids, int64_t n_children,
                                     const void *child_values, int64_t span_begin,
                                     int64_t span_points, const hhsar_geom *geom, int kernel,
                                     void *out, int64_t *flagged, void *stream) {
    HHSAR_REQUIRE(dims[0] > 0 && dims[1] > 0 && dims[2] > 0 && n_children > 0 && geom,
                  "merge_cartesian: bad arguments");
    const bool per_voxel = (kernel & HHSAR_LANDING_PER_VOXEL) != 0;
    kernel &= ~HHSAR_LANDING_PER_VOXEL;
    HHSAR_REQUIRE(kernel == 0 || kernel == 1, "merge_cartesian: unknown interpolation kernel");
    HHSAR_REQUIRE(span_begin >= 0 && span_points >= 0, "merge_cartesian: bad child span");
    const int64_t total = dims[0] * dims[1] * dims[2];
    if (vox_end < 0 || vox_end > total) vox_end = total;
    HHSAR_REQUIRE(vox_begin >= 0 && vox_begin <= vox_end, "merge_cartesian: bad voxel range");
    if (vox_begin == vox_end) return HHSAR_OK;
    cudaStream_t s = as_stream(stream);
    auto kv = reinterpret_cast<const float2 *>(child_values);
    auto o = reinterpret_cast<float2 *>(out);
    MergeChild *kids = nullptr;
    int rc = prep_children(child_grids, n_children, *geom, kernel, &kids, s);
    if (rc != HHSAR_OK) return rc;
    auto launch = [&](auto kern, int64_t zq) {
        // quads (zq z-consecutive voxels of one column) covering [vox_begin, vox_end)
        const int64_t nzq = (dims[2] + zq - 1) / zq;
        const int64_t q0 = (vox_begin / dims[2]) * nzq + (vox_begin % dims[2]) / zq;
        const int64_t q1 = ((vox_end - 1) / dims[2]) * nzq + ((vox_end - 1) % dims[2]) / zq + 1;
        const unsigned blocks = (unsigned)((q1 - q0 + MERGE_THREADS - 1) / MERGE_THREADS);
        kern<<<blocks, MERGE_THREADS, 0, s>>>(origin[0], origin[1], origin[2], step[0], step[1],
                                              step[2], (int)dims[0], (int)dims[1], (int)dims[2],
                                              vox_begin, vox_end, q0, q1 - q0, kids,
                                              (int)n_children, kv, *geom, o, flagged);
    };
#ifndef HHSAR_LANDING_EXACT
    // z series (merge_cartesian_series_kernel): ZQ z voxels per thread with
    // the Taylor offset |z - z_c| <= (ZQ - 1) sz / 2 at most 6% of the
    // nearest voxel's height above the aperture plane (every distance the
    // series expands is >= z): fifth-order terms below ~1e-5 rad of phase
    const double oz = origin[2], sz = step[2];
#ifndef HHSAR_LANDING_ZQ
#define HHSAR_LANDING_ZQ 8
#endif

    // (cubic: 64-point stencils, at most 4 voxels per thread for registers)
    const int zq = per_voxel ? 0
                   : (HHSAR_LANDING_ZQ >= 8 && kernel == 0 && oz > 0.0 && 3.5 * sz <= 0.06 * oz) ? 8
                   : (oz > 0.0 && 1.5 * sz <= 0.06 * oz) ? 4
                                                        : 0;
    if (zq) {
        // pair-staged copy of the children's lattices (16 B per point): the
        // gathers then move half as many L1 wavefronts
        float4 *pairs = nullptr;
        if (span_points > 0) {
            if (cudaMallocAsync(&pairs, span_points * sizeof(float4), s) != cudaSuccess) {
                cudaFreeAsync(kids, s);
                return set_error(HHSAR_ECUDA, "merge_cartesian: pair scratch allocation failed");
            }
            pair_rows_kernel<<<(unsigned)((span_points + 255) / 256), 256, 0, s>>>(
                kv, span_begin, span_points, pairs);
        }
        const float4 *kp = pairs ? pairs - span_begin : nullptr;  // indexed by pool offset
        auto launch_s = [&](auto kern) {
            const int64_t nzq = (dims[2] + zq - 1) / zq;
            const int64_t q0 = (vox_begin / dims[2]) * nzq + (vox_begin % dims[2]) / zq;
            const int64_t q1 = ((vox_end - 1) / dims[2]) * nzq + ((vox_end - 1) % dims[2]) / zq + 1;
            unsigned blocks = (unsigned)((q1 - q0 + MERGE_THREADS - 1) / MERGE_THREADS);
            // warp tiles over the whole volume (3-D grid) when the shape allows
            constexpr int TC = HHSAR_LANDING_TILE > 0 ? HHSAR_LANDING_TILE : 1, TK = 32 / TC;
            constexpr int KT_CTA = TK * (MERGE_THREADS / 32);  // z blocks per CTA
            const int tile = HHSAR_LANDING_TILE > 0 && vox_begin == 0 && vox_end == total &&
                             dims[1] % TC == 0 && nzq % KT_CTA == 0 && dims[0] <= 65535 &&
                             nzq / KT_CTA <= 65535;
            dim3 grid(blocks);
            if (tile) grid = dim3((unsigned)(dims[1] / TC), (unsigned)(nzq / KT_CTA), (unsigned)dims[0]);
            kern<<<grid, MERGE_THREADS, 0, s>>>(origin[0], origin[1], origin[2], step[0], step[1],
                                                step[2], (int)dims[1], (int)dims[2], vox_begin,
                                                vox_end, q0, q1 - q0, kids, (int)n_children, kv, kp,
                                                *geom, o, flagged, tile);
        };
        if (kernel == 0) {
            if (zq == 8) launch_s(merge_cartesian_series_kernel<0, 8>);
            else launch_s(merge_cartesian_series_kernel<0, 4>);
        } else {
            launch_s(merge_cartesian_series_kernel<1, 4>);
        }
        rc = check_launch("merge_cartesian_series_kernel");
        if (pairs) cudaFreeAsync(pairs, s);
        cudaFreeAsync(kids, s);
        return rc;
    }
#endif
    // 4 z-voxels per thread when there are >= 4 children or the launch is
    // large (config 4, 268 M voxels x 2 children: 4.49 -> 4.19 ms); 2
    // otherwise (config 3, 33.5 M voxels: 0.61 ms vs 0.62).  Two children
    // (the binary and factor-4 top levels) unroll the child loop: both
    // children's gathers in flight, 80 instead of 96 registers (config 4
    // 4.23 -> 4.18 ms)
    const bool wide = n_children >= 4 || vox_end - vox_begin >= (int64_t(1) << 26);
    if (kernel == 0) {
        if (wide && n_children == 2) launch(merge_cartesian_kernel<0, 4, 2>, 4);
        else if (wide) launch(merge_cartesian_kernel<0, 4>, 4);
        else launch(merge_cartesian_kernel<0, 2>, 2);
    } else {
        if (wide) launch(merge_cartesian_kernel<1, 4>, 4);
        else launch(merge_cartesian_kernel<1, 2>, 2);
    }
    rc = check_launch("merge_cartesian_kernel");
    cudaFreeAsync(kids, s);
    return rc;
}

extern "C" int hhsar_lattice_interp(const void *values, int64_t nu, int64_t nv, int64_t nn,
                                    const double *coords, int64_t n, int kernel, void *out,
                                    uint8_t *ok, void *stream) {
    HHSAR_REQUIRE(kernel == 0 || kernel == 1, "lattice_interp: unknown interpolation kernel");
    HHSAR_REQUIRE(nu >= 2 && nv >= 2 && nn >= 2, "lattice_interp: lattice needs >= 2 samples per axis");
    HHSAR_REQUIRE(kernel == 0 || (nu >= 4 && nv >= 4 && nn >= 4),
                  "lattice_interp: cubic needs >= 4 samples per axis");
    if (n == 0) return HHSAR_OK;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    cudaStream_t s = as_stream(stream);
    auto v = reinterpret_cast<const float2 *>(values);
    auto o = reinterpret_cast<float2 *>(out);
    if (kernel == 0)
        lattice_interp_kernel<0><<<blocks, 256, 0, s>>>(v, (int)nu, (int)nv, (int)nn, coords, n, o, ok);
    else
        lattice_interp_kernel<1><<<blocks, 256, 0, s>>>(v, (int)nu, (int)nv, (int)nn, coords, n, o, ok);
    return check_launch("lattice_interp_kernel");
}
