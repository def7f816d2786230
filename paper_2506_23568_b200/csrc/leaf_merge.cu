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
    const int su = C.nv * C.nn;  // lattices hold < 2^31 points (int32 dims product)
    const float2 *base = vals + C.offset;
    float2 acc = make_float2(0.f, 0.f);
    if (KERNEL == 0) {
        // trilinear as nested lerps along n, v, u on (re, im) pairs: one
        // FADD2 + one FFMA2 per lerp, no weight products
        const float2 *b = base + ((iu * C.nv + iv) * C.nn + iw);
        f2x r[2][2];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int bb = 0; bb < 2; ++bb) {
                const float2 *row = b + a * su + bb * C.nn;
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
    out = acc;
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
                                     const void *child_values, const hhsar_geom *geom, int kernel,
                                     void *out, int64_t *flagged, void *stream) {
    HHSAR_REQUIRE(dims[0] > 0 && dims[1] > 0 && dims[2] > 0 && n_children > 0 && geom,
                  "merge_cartesian: bad arguments");
    HHSAR_REQUIRE(kernel == 0 || kernel == 1, "merge_cartesian: unknown interpolation kernel");
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
