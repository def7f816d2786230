// Subimage lattice construction for every subarray of every level in two
// launches (reference: ffbp.py:179-307 build_subimage_grid, the Newton loop
// _kernels.py:255-351, and the leaf delay mask ffbp.py:320-335).
//
// hhsar_grid_plan: one CTA per grid.  Element bbox from the leaf boxes, the
// 125-point boundary map, and every integer decision of the lattice (counts,
// u/v trimming, near band, core box) in bit-exact float64 (no FMA, same
// operation order as numpy), so dims/origin/masks equal the reference's.
//
// hhsar_grid_newton: one thread per (u, v) column, marching along n with the
// reference's warm starts (ffbp.py:274-282).  Columns outside the near band
// are skipped (all their points are masked whatever Newton returns) and the
// march stops after the last near plane -- exact pruning, SURVEY G3.
#include <cfloat>

#include "common.cuh"

#include <cstdlib>

namespace hhsar {

constexpr int PLAN_THREADS = 128;

// ---- damped Newton (_kernels.py:255-351) ------------------------------------
struct NewtonGeom {
    double ext[4];
    double gap, c_uv, c_nhi, c_nlo;
};

// ---- one Newton iteration, SFU-seeded float64 reciprocal square roots ---------
// Every distance the iteration needs is d = a * rsqrt(a) with a the squared
// distance; its reciprocal (Jacobian) is rsqrt(a) itself, so the 8 sqrt + 9
// divisions of the textbook form become 9 rsqrt + 1 reciprocal (rsqrt_d /
// rcp_d in common.cuh: fp32 SFU seed + one float64 Newton step, relative
// error ~1e-13; the residual test is on (u, v, n) values of O(10-100) against
// tol = 1e-9, so this rounding is ~1e-11 of noise, far below the tolerance).

// Returns 1 when the residual at (x, y, z) is within tol (converged), 2 when
// the reference would give up here (rad <= 0, a zero distance, singular
// Jacobian), 0 after taking one damped step (same formulas as
// _kernels.py:277-340).
__device__ __forceinline__ int newton_iteration(const NewtonGeom &G, double tu, double tv,
                                                double tn, double &x, double &y, double &z,
                                                double tol, double max_step2, double max_step,
                                                double z_floor) {
    const double xmn = G.ext[0], xmx = G.ext[1], ymn = G.ext[2], ymx = G.ext[3];
    // clamps, zero test and convergence test written with comparisons: the
    // float64 fmin / fmax of sm_100 cost ~8 instructions each (DSETP.MIN +
    // NaN-handling selects), ~40% of an iteration in this form.  Results are
    // those of fmin / fmax (NaN operands ignored) for every input.
    const double xc = x > xmn ? x : xmn, yc = y > ymn ? y : ymn;  // fmax(x, lo): NaN -> lo
    const double x0 = xc < xmx ? xc : xmx, y0 = yc < ymx ? yc : ymx;
    const double z2 = z * z;
    const double ax = x - xmn, bx = x - xmx, ay = y - ymn, by = y - ymx;
    const double yd = y - y0, xd = x - x0;
    const double yy = yd * yd, xx = xd * xd;
    const double ax2 = ax * ax, bx2 = bx * bx, ay2 = ay * ay, by2 = by * by;
    const double a_u1 = ax2 + yy + z2, a_u2 = bx2 + yy + z2;
    const double a_v1 = xx + ay2 + z2, a_v2 = xx + by2 + z2;
    const double a_e1 = ax2 + ay2 + z2, a_e2 = ax2 + by2 + z2;
    const double a_e3 = bx2 + ay2 + z2, a_e4 = bx2 + by2 + z2;
    // fmin over the eight == 0  <=>  some (non-NaN) value == 0
    if ((a_u1 == 0.0) | (a_u2 == 0.0) | (a_v1 == 0.0) | (a_v2 == 0.0) | (a_e1 == 0.0) |
        (a_e2 == 0.0) | (a_e3 == 0.0) | (a_e4 == 0.0))
        return 2;
    const double i1 = rsqrt_d(a_u1), i2 = rsqrt_d(a_u2), i3 = rsqrt_d(a_v1), i4 = rsqrt_d(a_v2);
    const double f1 = rsqrt_d(a_e1), f2 = rsqrt_d(a_e2), f3 = rsqrt_d(a_e3), f4 = rsqrt_d(a_e4);
    const double r = a_e1 * f1 + a_e2 * f2 + a_e3 * f3 + a_e4 * f4;
    const double rad = r * r - G.gap;
    if (rad <= 0.0) return 2;
    const double irad = rsqrt_d(rad);
    const double sq = rad * irad;
    const double ru = G.c_uv * (a_u1 * i1 - a_u2 * i2) - tu;
    const double rv = G.c_uv * (a_v1 * i3 - a_v2 * i4) - tv;
    const double rn = G.c_nhi * sq - G.c_nlo * r - tn;
    // fmax(|ru|, |rv|, |rn|) <= tol with fmax's NaN rule (a NaN operand is
    // ignored; all three NaN -> NaN -> false)
    if (!(fabs(ru) > tol) & !(fabs(rv) > tol) & !(fabs(rn) > tol) &
        !((ru != ru) & (rv != rv) & (rn != rn)))
        return 1;
    const double ja = G.c_uv * (ax * i1 - bx * i2);
    const double jb = G.c_uv * (yd * (i1 - i2));
    const double jc = G.c_uv * (z * (i1 - i2));
    const double jd = G.c_uv * (xd * (i3 - i4));
    const double je = G.c_uv * (ay * i3 - by * i4);
    const double jf = G.c_uv * (z * (i3 - i4));
    const double fac = G.c_nhi * (r * irad) - G.c_nlo;
    const double jg = fac * (ax * (f1 + f2) + bx * (f3 + f4));
    const double jh = fac * (ay * (f1 + f3) + by * (f2 + f4));
    const double ji = fac * (z * (f1 + f2 + f3 + f4));
    const double m0 = je * ji - jf * jh, m1 = jd * ji - jf * jg, m2 = jd * jh - je * jg;
    const double det = ja * m0 - jb * m1 + jc * m2;
    if (fabs(det) < 1e-30) return 2;
    const double idet = rcp_d(det);
    double sx = (ru * m0 - jb * (rv * ji - jf * rn) + jc * (rv * jh - je * rn)) * idet;
    double sy = (ja * (rv * ji - jf * rn) - ru * m1 + jc * (jd * rn - rv * jg)) * idet;
    double sz = (ja * (je * rn - rv * jh) - jb * (jd * rn - rv * jg) + ru * m2) * idet;
    if (max_step > 0.0) {
        const double sn2 = sx * sx + sy * sy + sz * sz;
        if (sn2 > max_step2) {
            const double sc = max_step * rsqrt_d(sn2);
            sx *= sc;
            sy *= sc;
            sz *= sc;
        }
    }
    x -= sx;
    y -= sy;
    z -= sz;
    if (z < z_floor) z = z_floor;
    return 0;
}

// ---- leaf boxes ----------------------------------------------------------------
template <int N>
__device__ void block_minmax(double (&mn)[N], double (&mx)[N]) {
    __shared__ double s_mn[N][PLAN_THREADS / 32], s_mx[N][PLAN_THREADS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[k] = fmin(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
            mx[k] = fmax(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
        }
        if (lane == 0) {
            s_mn[k][wid] = mn[k];
            s_mx[k][wid] = mx[k];
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < N; ++k) {
        mn[k] = s_mn[k][0];
        mx[k] = s_mx[k][0];
        for (int w = 1; w < PLAN_THREADS / 32; ++w) {
            mn[k] = fmin(mn[k], s_mn[k][w]);
            mx[k] = fmax(mx[k], s_mx[k][w]);
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(PLAN_THREADS)
leaf_boxes_kernel(const double *__restrict__ el, const int64_t *__restrict__ bounds,
                  double *__restrict__ box) {
    const int64_t l = blockIdx.x;
    double mn[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, mx[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
    for (int64_t i = bounds[l] + threadIdx.x; i < bounds[l + 1]; i += PLAN_THREADS)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            mn[a] = fmin(mn[a], el[3 * i + a]);
            mx[a] = fmax(mx[a], el[3 * i + a]);
        }
    block_minmax<3>(mn, mx);
    if (threadIdx.x == 0)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            box[6 * l + a] = mn[a];
            box[6 * l + 3 + a] = mx[a];
        }
}

// ---- lattice plan (ffbp.py:226-304) ---------------------------------------------
__global__ void __launch_bounds__(PLAN_THREADS)
grid_plan_kernel(hhsar_grid_desc *__restrict__ grids, const double *__restrict__ leaf_box,
                 const double *__restrict__ boundary, int n_b, hhsar_geom g,
                 int32_t *__restrict__ status) {
    hhsar_grid_desc &D = grids[blockIdx.x];
    // element bbox over the grid's leaves (exact: min/max)
    double mn[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, mx[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
    for (int64_t l = D.leaf_lo + threadIdx.x; l < D.leaf_hi; l += PLAN_THREADS)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            mn[a] = fmin(mn[a], leaf_box[6 * l + a]);
            mx[a] = fmax(mx[a], leaf_box[6 * l + 3 + a]);
        }
    block_minmax<3>(mn, mx);
    const double ext[4] = {mn[0], mx[0], mn[1], mx[1]};
    // forward map of the region's boundary lattice -> lo, hi (ffbp.py:237-240)
    double lo[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, hi[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
    bool bad = false;
    for (int i = threadIdx.x; i < n_b; i += PLAN_THREADS) {
        double uvn[3];
        bad |= !llt_exact(ext, g, boundary[3 * i], boundary[3 * i + 1], boundary[3 * i + 2], uvn);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo[a] = fmin(lo[a], uvn[a]);
            hi[a] = fmax(hi[a], uvn[a]);
        }
    }
    if (bad) atomicExch(status, 1);
    block_minmax<3>(lo, hi);
    if (threadIdx.x != 0) return;

    const double step = g.step;
    const double padstep = xmul((double)g.pad, step);
    double origin[3];
    int cnt[3];
    for (int a = 0; a < 3; ++a) {
        origin[a] = xsub(lo[a], padstep);
        cnt[a] = (int)ceil(xdiv(xsub(hi[a], lo[a]), step)) + 1 + 2 * g.pad;
    }
    // u/v trimming (ffbp.py:248-257)
    const double limit[2] = {xmul(g.c_uv, xsub(ext[1], ext[0])), xmul(g.c_uv, xsub(ext[3], ext[2]))};
    for (int a = 0; a < 2; ++a) {
        const double thr = xadd(limit[a], xmul(2.0, step));
        int first = -1, last = -1;
        for (int i = 0; i < cnt[a]; ++i) {
            const double plane = xadd(origin[a], xmul(step, (double)i));
            if (fabs(plane) < thr) {
                if (first < 0) first = i;
                last = i;
            }
        }
        const bool any = first >= 0, all = any && first == 0 && last == cnt[a] - 1 &&
                                           (last - first + 1) == cnt[a];
        // "all" must also mean no gap; keep is contiguous (|plane| is unimodal)
        if (any && !all) {
            origin[a] = xadd(origin[a], xmul((double)first, step));
            cnt[a] = last - first + 1;
        }
    }
    const double rlo[3] = {g.region[0], g.region[2], g.region[4]};
    const double rhi[3] = {g.region[1], g.region[3], g.region[5]};
    const double eps = xmul(1e-9, step);
    const double two_step = xmul(2.0, step);
    for (int a = 0; a < 3; ++a) {
        const double extent = xsub(rhi[a], rlo[a]);
        // shadow = 3.0 * GRID_PAD * step * extent / max(hi - lo, 1e-12)
        const double shadow = xdiv(xmul(xmul(6.0, step), extent), fmax(xsub(hi[a], lo[a]), 1e-12));
        const double slack = xadd(xmul(g.margin, extent), shadow);
        D.slack_lo[a] = xsub(rlo[a], slack);
        D.slack_hi[a] = xadd(rhi[a], slack);
        const double near_a = xsub(xsub(lo[a], two_step), eps);
        const double near_b = xadd(xadd(hi[a], two_step), eps);
        const double img_a = xsub(lo[a], eps), img_b = xadd(hi[a], eps);
        int n0 = -1, n1 = -2, c0 = -1, c1 = -1;
        for (int i = 0; i < cnt[a]; ++i) {
            const double t = xadd(origin[a], xmul(step, (double)i));
            if (t >= near_a && t <= near_b) {
                if (n0 < 0) n0 = i;
                n1 = i;
            }
            if (t >= img_a && t <= img_b) {
                if (c0 < 0) c0 = i;
                c1 = i;
            }
        }
        if (n0 < 0) n0 = 0;            // empty band: lo > hi
        if (c0 < 0) { c0 = 0; c1 = cnt[a] - 1; }  // np.argmax of all-False
        D.near_lo[a] = n0;
        D.near_hi[a] = n1;
        D.core_lo[a] = c0;
        D.core_hi[a] = c1;
        D.origin[a] = origin[a];
        D.dims[a] = cnt[a];
        D.lo[a] = lo[a];
        D.hi[a] = hi[a];
        D.box[a] = mn[a];
        D.box[3 + a] = mx[a];
        if (a < 2) {
            // Active columns: the near band intersected with the reachable
            // targets.  |u| < (k_max/pi) dx for every point with z > 0
            // (triangle inequality on du1 - du2; v likewise), so a column with
            // |tu| >= (k_max/pi) dx + 2 tol cannot converge on any plane: all
            // its points fail -- which also keeps its warm-start chain at the
            // region centre -- and are masked without running Newton.  These
            // are the u/v planes the reference keeps just beyond the limit
            // (ffbp.py:248-257).  Both sets are index intervals.
            const double lim = g.c_uv * (ext[2 * a + 1] - ext[2 * a]) + 2.0 * g.tol;
            int a0 = -1, a1 = -2;
            for (int i = n0; i <= n1; ++i) {
                const double t = xadd(origin[a], xmul(step, (double)i));
                if (fabs(t) < lim) {
                    if (a0 < 0) a0 = i;
                    a1 = i;
                }
            }
            if (a0 < 0) a0 = 0;
            D.act_lo[a] = a0;
            D.act_hi[a] = a1;
        }
    }
    for (int k = 0; k < 4; ++k) D.ext[k] = ext[k];
}

// ---- Newton columns -------------------------------------------------------------
// Work list = the active columns only (desc.act_* rectangle, see
// grid_plan_kernel): columns outside the near band are masked whatever
// Newton returns (ffbp.py:294-301) and unreachable ones provably fail, so
// neither is launched (the caller zeroed `valid`).  Within a column the
// reference marches the n planes in order, warm-starting plane w + 1 from
// plane w's solution when plane w converged and from the region centre
// otherwise (ffbp.py:274-282).
//
// * light columns: persistent kernel with PER-LANE work fetching -- every
//   lane runs its own (column, plane, iteration) state machine and grabs the
//   next column from a global counter when done;
// * heavy columns: segments of planes solved speculatively in parallel, then
//   a fix-up pass in the reference's order (below).
constexpr int NEWTON_THREADS = 128;
constexpr int HEAVY_MAXP = 64;  // planes per heavy column held in shared memory
constexpr int64_t NEWTON_SPEC2_MAX_COLS = 131072;  // speculative continuations up to this size
constexpr int SPEC_DEPTH = 8;  // warm planes a speculative chain runs past its centre start

__device__ __forceinline__ int grid_of_column(const hhsar_grid_desc *__restrict__ grids,
                                              int n_grids, const int32_t *__restrict__ block_grid,
                                              unsigned long long c) {
    if (block_grid) {
        int g2 = block_grid[c >> 7];
        while (g2 + 1 < n_grids && (unsigned long long)grids[g2 + 1].col_offset <= c) ++g2;
        return g2;
    }
    int lo = 0, hi = n_grids - 1;  // last grid whose col_offset <= c (empty grids share offsets)
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((unsigned long long)grids[mid].col_offset <= c) lo = mid; else hi = mid - 1;
    }
    return lo;
}

struct Column {
    int gi, iu, iv;
    double tu, tv;
};

__device__ __forceinline__ Column decode_in_grid(const hhsar_grid_desc *__restrict__ grids,
                                                 int gi, const hhsar_geom &g,
                                                 unsigned long long c) {
    Column q;
    q.gi = gi;
    const hhsar_grid_desc &D = grids[q.gi];
    const int k = (int)((int64_t)c - D.col_offset);
    const int wv = D.act_hi[1] - D.act_lo[1] + 1;
    const int ku = k / wv;
    q.iu = D.act_lo[0] + ku;
    q.iv = D.act_lo[1] + (k - ku * wv);
    q.tu = xadd(D.origin[0], xmul(g.step, (double)q.iu));
    q.tv = xadd(D.origin[1], xmul(g.step, (double)q.iv));
    return q;
}

__device__ __forceinline__ Column decode_column(const hhsar_grid_desc *__restrict__ grids,
                                                int n_grids, const int32_t *block_grid,
                                                const hhsar_geom &g, unsigned long long c) {
    return decode_in_grid(grids, grid_of_column(grids, n_grids, block_grid, c), g, c);
}

// per-column record written once by grid_newton_heavy_list_kernel: the
// column's grid index, bit 31 = heavy
constexpr int32_t HEAVY_BIT = (int32_t)0x80000000;

__device__ __forceinline__ bool column_is_heavy(const hhsar_grid_desc &D, const hhsar_geom &g,
                                                double tu, double tv) {
    const double qu = tu / (g.c_uv * (D.ext[1] - D.ext[0]));
    const double qv = tv / (g.c_uv * (D.ext[3] - D.ext[2]));
    return qu * qu + qv * qv >= 1.0 && D.near_hi[2] + 1 <= HEAVY_MAXP;
}

__device__ __forceinline__ void column_geom(const hhsar_grid_desc &D, const hhsar_geom &g,
                                            NewtonGeom &G) {
    G.c_uv = g.c_uv;
    G.c_nhi = g.c_nhi;
    G.c_nlo = g.c_nlo;
    for (int q = 0; q < 4; ++q) G.ext[q] = D.ext[q];
    G.gap = box_gap_exact(D.ext);
}

// One plane: damped Newton from (x, y, z) (z floored first) until converged,
// given up, or max_iter iterations; returns the newton_iteration status.
__device__ __forceinline__ int solve_plane(const NewtonGeom &G, const hhsar_geom &g, double tu,
                                           double tv, double tn, double &x, double &y, double &z,
                                           int &it) {
    const double max_step2 = g.max_step * g.max_step;
    if (z < g.z_floor) z = g.z_floor;
    it = 0;
    int st = 0;
    while (st == 0 && it < g.max_iter) {
        ++it;
        st = newton_iteration(G, tu, tv, tn, x, y, z, g.tol, max_step2, g.max_step, g.z_floor);
    }
    return st;
}

__device__ __forceinline__ double plane_target(const hhsar_grid_desc &D, const hhsar_geom &g,
                                               int w) {
    return xadd(D.origin[2], xmul(g.step, (double)w));
}

// Masks and counters of plane w of a column once its solve is final:
// containment (slack) -> valid point, leaf delay window (ffbp.py:320-335),
// core counts; positions of contained points.
__device__ __forceinline__ void finish_plane(const hhsar_grid_desc &D, const hhsar_geom &g, int w,
                                             bool ok, double x, double y, double z, bool core_uv,
                                             int64_t base, uint8_t *__restrict__ valid,
                                             double *__restrict__ positions, unsigned (&acc)[6]) {
    // every descriptor field this needs is loaded up front (independent
    // loads in flight together; no short-circuit chain of dependent loads)
    const int near_lo = D.near_lo[2], is_leaf = D.is_leaf, core_lo = D.core_lo[2],
              core_hi = D.core_hi[2];
    const double sl0 = D.slack_lo[0], sl1 = D.slack_lo[1], sl2 = D.slack_lo[2];
    const double sh0 = D.slack_hi[0], sh1 = D.slack_hi[1], sh2 = D.slack_hi[2];
    const double b0 = D.box[0], b1 = D.box[1], b2 = D.box[2], b3 = D.box[3], b4 = D.box[4],
                 b5 = D.box[5];
    if (w < near_lo) return;
    const bool pre = ok & (x >= sl0) & (x <= sh0) & (y >= sl1) & (y <= sh1) & (z >= sl2) &
                     (z <= sh2);
    bool post = pre;
    if (pre && is_leaf) {
        // 2 * max corner distance / c <= window_hi (ffbp.py:320-330).  The
        // farthest of the 8 corners takes, per axis, the bound farther from
        // the point; rounded subtraction, squaring, addition and sqrt are all
        // monotone, so its rounded distance IS the reference's max over the 8
        // (bit-exact, 1 sqrt not 8).
        const double ex0 = xsub(x, b0), ex1 = xsub(x, b3);
        const double ey0 = xsub(y, b1), ey1 = xsub(y, b4);
        const double ez0 = xsub(z, b2), ez1 = xsub(z, b5);
        const double fx = fabs(ex0) >= fabs(ex1) ? ex0 : ex1;
        const double fy = fabs(ey0) >= fabs(ey1) ? ey0 : ey1;
        const double fz = fabs(ez0) >= fabs(ez1) ? ez0 : ez1;
        const double s2 = xadd(xadd(xsq(fx), xsq(fy)), xsq(fz));
        // decided on the square unless within 1e-12 of the limit (the exact
        // sqrt / divide round to < 3e-16 relative, so outside that band the
        // reference's comparison cannot come out differently)
        const double lim = 0.5 * HHSAR_C_LIGHT * g.window_hi, lim2 = lim * lim;
        if (s2 < lim2 * (1.0 - 1e-12)) {
            post = true;
        } else if (s2 > lim2 * (1.0 + 1e-12)) {
            post = false;
        } else {
            const double dmax = xsqrt(s2);
            post = xdiv(xmul(2.0, dmax), HHSAR_C_LIGHT) <= g.window_hi;
        }
    }
    const bool in_core = core_uv & (w >= core_lo) & (w <= core_hi);
    acc[0] += pre;
    acc[1] += pre && in_core;
    acc[2] += post;
    acc[3] += post && in_core;
    if (post) valid[base + w] = 1;
    if (pre) {
        double *pp = positions + 3 * (base + w);
        pp[0] = x;
        pp[1] = y;
        pp[2] = z;
    }
}

__device__ __forceinline__ void flush_stats(int64_t *__restrict__ stats, int gi,
                                            unsigned (&acc)[6]) {
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        if (acc[q])
            atomicAdd((unsigned long long *)(stats + (int64_t)gi * HHSAR_GRID_STATS + q),
                      (unsigned long long)acc[q]);
        acc[q] = 0;
    }
}

// Heavy columns -- (u, v) outside the far-field ellipse (tu/U)^2 + (tv/V)^2
// < 1, U = c_uv dx, V = c_uv dy -- fail plane after plane (config 3: 6% of
// the columns, ~800 iterations each against ~80, 39% of all iterations), and
// a failed plane restarts the next one from the region centre, so their
// chains are mostly broken.  grid_newton_heavy_list_kernel collects them;
// grid_newton_kernel solves every heavy plane independently from the centre
// (one task per plane, started before the light columns) and stores the
// speculative (ok, iterations) in `valid`, positions in `positions`;
// grid_newton_fixup_kernel then walks each heavy column in the reference's
// order and re-solves, warm-started, exactly the planes whose predecessor
// converged (the reference did not restart those from the centre).  Every
// plane ends with the reference's start point, so results and iteration
// counts are unchanged; all tasks are short, so the persistent kernel can
// run at full occupancy without a long tail.
__device__ __forceinline__ uint8_t spec_code(bool ok, int it) {
    return (uint8_t)((ok ? 0x80 : 0) | (it & 0x7f));  // it <= max_iter <= 126 (checked at entry)
}

__global__ void grid_newton_heavy_list_kernel(const hhsar_grid_desc *__restrict__ grids,
                                              int n_grids, int64_t n_cols,
                                              const int32_t *__restrict__ block_grid,
                                              hhsar_geom g, int32_t *__restrict__ heavy,
                                              unsigned long long *__restrict__ n_heavy,
                                              int32_t *__restrict__ col_grid) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool h = false;
    if (c < n_cols) {
        const Column q = decode_column(grids, n_grids, block_grid, g, (unsigned long long)c);
        h = column_is_heavy(grids[q.gi], g, q.tu, q.tv);
        col_grid[c] = q.gi | (h ? HEAVY_BIT : 0);
    }
    const unsigned m = __ballot_sync(0xffffffffu, h);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    unsigned long long b0 = 0;
    if (lane == __ffs(m) - 1) b0 = atomicAdd(n_heavy, (unsigned long long)__popc(m));
    b0 = __shfl_sync(0xffffffffu, b0, __ffs(m) - 1);
    if (h) heavy[b0 + __popc(m & ((1u << lane) - 1u))] = (int32_t)c;
}

// SPEC2 (heavy phase, small problems): a heavy plane s whose centre start
// converged goes on warm through the next planes -- s+1 from s, s+2 from
// s+1, ... while they converge, up to SPEC_DEPTH planes -- and stores plane
// s+d in spec2_* slot [heavy index][plane s+d][d-1].  When the reference's
// run of converged planes starts at s (s-1 failed, so s itself started
// from the centre), that chain IS the reference's sequence of solves, so
// the in-order fix-up only solves planes deeper than SPEC_DEPTH into a run.
template <bool SPEC2>
__global__ void __launch_bounds__(NEWTON_THREADS)
grid_newton_kernel(const hhsar_grid_desc *__restrict__ grids, int n_grids, int64_t n_cols,
                   const int32_t *__restrict__ block_grid, hhsar_geom g,
                   double *__restrict__ positions, uint8_t *__restrict__ valid,
                   int64_t *__restrict__ stats, unsigned long long *__restrict__ counter,
                   const int32_t *__restrict__ heavy, const unsigned long long *__restrict__ n_heavy_p,
                   int phase, const int32_t *__restrict__ col_grid, double *__restrict__ spec2_pos,
                   uint8_t *__restrict__ spec2_code, int64_t spec2_cap) {
    NewtonGeom G;
    int gi = -1, acc_gi = -1, w = 0, w_end = 0, it = 0, iu = 0, iv = 0;
    int64_t base = 0;  // lattice index of plane 0 of the current column
    bool have = false, core_uv = false, spec = false, warm2 = false;
    int64_t hslot = 0;  // SPEC2: heavy index * HEAVY_MAXP
    int depth = 0;      // SPEC2: warm planes past the centre start
    double tu = 0, tv = 0, tn = 0, x = 0, y = 0, z = 0;
    const double max_step2 = g.max_step * g.max_step;
    // phase 0: heavy (column, plane) slots only; phase 1: light columns only
    const unsigned long long n_spec = phase == 0 ? *n_heavy_p * HEAVY_MAXP : 0;
    const unsigned long long n_light = phase == 0 ? 0 : (unsigned long long)n_cols;
    unsigned acc[6] = {0, 0, 0, 0, 0, 0};
    auto start_plane = [&](const hhsar_grid_desc &D, double sx, double sy, double sz) {
        tn = plane_target(D, g, w);
        x = sx;
        y = sy;
        z = sz > g.z_floor ? sz : g.z_floor;
        it = 0;
    };
    while (true) {
        if (!have) {
            // first the heavy planes (one task each), then the light columns
            const unsigned long long t = atomicAdd(counter, 1ull);
            if (t >= n_spec + n_light) break;
            spec = t < n_spec;
            const unsigned long long c =
                spec ? (unsigned long long)heavy[t / HEAVY_MAXP] : t - n_spec;
            const int32_t rec = __ldg(col_grid + c);
            if (!spec && (rec & HEAVY_BIT)) continue;  // solved plane by plane in phase 0
            const Column q = decode_in_grid(grids, rec & ~HEAVY_BIT, g, c);
            const hhsar_grid_desc &D = grids[q.gi];
            const int wend_col = D.near_hi[2] + 1;
            if (spec) {
                w = (int)(t % HEAVY_MAXP);
                if (w >= wend_col) continue;
                w_end = w + 1;
                if constexpr (SPEC2) {
                    hslot = (int64_t)(t / HEAVY_MAXP) * HEAVY_MAXP;
                    warm2 = false;
                    depth = 0;
                    // the warm continuation needs the next planes and a slot
                    if (w + 1 < wend_col && (int64_t)(t / HEAVY_MAXP) < spec2_cap)
                        w_end = min(wend_col, w + 1 + SPEC_DEPTH);
                }
            } else {
                w = 0;
                w_end = wend_col;
                if (q.gi != acc_gi) {
                    if (acc_gi >= 0) flush_stats(stats, acc_gi, acc);
                    acc_gi = q.gi;
                }
            }
            gi = q.gi;
            iu = q.iu;
            iv = q.iv;
            tu = q.tu;
            tv = q.tv;
            base = D.offset + ((int64_t)iu * D.dims[1] + iv) * D.dims[2];
            core_uv = iu >= D.core_lo[0] && iu <= D.core_hi[0] && iv >= D.core_lo[1] &&
                      iv <= D.core_hi[1];
            column_geom(D, g, G);
            have = w < w_end;
            if (have) start_plane(D, g.center[0], g.center[1], g.center[2]);
            continue;
        }
        ++it;
        const int st = newton_iteration(G, tu, tv, tn, x, y, z, g.tol, max_step2, g.max_step,
                                        g.z_floor);
        if (st == 0 && it < g.max_iter) continue;
        // plane w finished: masks, counters, warm start for plane w + 1
        const hhsar_grid_desc &D = grids[gi];
        const bool ok = st == 1;
        if (spec) {  // speculative: the fix-up kernel decides
            if (SPEC2 && warm2) {
                const int64_t slot = (hslot + w) * SPEC_DEPTH + (depth - 1);
                spec2_code[slot] = spec_code(ok, it);
                double *pp = spec2_pos + 3 * slot;
                pp[0] = x;
                pp[1] = y;
                pp[2] = z;
                if (ok && w + 1 < w_end) {  // the chain goes on
                    ++w;
                    ++depth;
                    start_plane(D, x, y, z);
                    continue;
                }
                have = false;
                continue;
            }
            valid[base + w] = spec_code(ok, it);
            double *pp = positions + 3 * (base + w);
            pp[0] = x;
            pp[1] = y;
            pp[2] = z;
            if (SPEC2 && ok && w + 1 < w_end) {  // continue warm on the next planes
                warm2 = true;
                depth = 1;
                ++w;
                start_plane(D, x, y, z);
                continue;
            }
            have = false;
            continue;
        }
        acc[4] += it;
        acc[5] += 1;
        finish_plane(D, g, w, ok, x, y, z, core_uv, base, valid, positions, acc);
        ++w;
        if (w >= w_end) {
            have = false;
            continue;
        }
        if (ok)
            start_plane(D, x, y, z);
        else
            start_plane(D, g.center[0], g.center[1], g.center[2]);
    }
    if (acc_gi >= 0) flush_stats(stats, acc_gi, acc);
}

__global__ void __launch_bounds__(NEWTON_THREADS)
grid_newton_fixup_kernel(const hhsar_grid_desc *__restrict__ grids, int n_grids,
                         const int32_t *__restrict__ block_grid, hhsar_geom g,
                         double *__restrict__ positions, uint8_t *__restrict__ valid,
                         int64_t *__restrict__ stats, const int32_t *__restrict__ heavy,
                         const unsigned long long *__restrict__ n_heavy_p,
                         const int32_t *__restrict__ col_grid,
                         const double *__restrict__ spec2_pos,
                         const uint8_t *__restrict__ spec2_code, int64_t spec2_cap) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)*n_heavy_p) return;
    const unsigned long long c = (unsigned long long)heavy[i];
    const Column q = decode_in_grid(grids, __ldg(col_grid + c) & ~HEAVY_BIT, g, c);
    const hhsar_grid_desc &D = grids[q.gi];
    NewtonGeom G;
    column_geom(D, g, G);
    const int w_end = D.near_hi[2] + 1;
    const int64_t base = D.offset + ((int64_t)q.iu * D.dims[1] + q.iv) * D.dims[2];
    const bool core_uv = q.iu >= D.core_lo[0] && q.iu <= D.core_hi[0] && q.iv >= D.core_lo[1] &&
                         q.iv <= D.core_hi[1];
    unsigned acc[6] = {0, 0, 0, 0, 0, 0};
    bool prev_ok = false;
    int run_start = 0;  // the plane the current run of converged planes started at
    double px = 0, py = 0, pz = 0;
    const bool has2 = spec2_code != nullptr && i < spec2_cap;
    for (int w = 0; w < w_end; ++w) {
        const uint8_t code = valid[base + w];
        double *pp = positions + 3 * (base + w);
        bool ok;
        int it;
        double x, y, z;
        const bool cold = !prev_ok;
        if (cold) run_start = w;
        const int depth = w - run_start;  // warm planes past the run's centre start
        const int64_t slot = ((int64_t)i * HEAVY_MAXP + w) * SPEC_DEPTH + (depth - 1);
        const uint8_t code2 = (has2 && !cold && depth <= SPEC_DEPTH) ? spec2_code[slot] : 0xff;
        if (cold) {  // the reference also started this plane from the centre
            ok = code & 0x80;
            it = code & 0x7f;
            x = pp[0];
            y = pp[1];
            z = pp[2];
        } else if (code2 != 0xff) {
            // the heavy phase's chain from this run's centre start already
            // solved this plane exactly as the reference does
            ok = code2 & 0x80;
            it = code2 & 0x7f;
            const double *q = spec2_pos + 3 * slot;
            x = q[0];
            y = q[1];
            z = q[2];
        } else {  // warm start from the converged predecessor
            x = px;
            y = py;
            z = pz;
            ok = solve_plane(G, g, q.tu, q.tv, plane_target(D, g, w), x, y, z, it) == 1;
        }
        valid[base + w] = 0;  // clear the speculative code; finish_plane sets 1
        acc[4] += it;
        acc[5] += 1;
        finish_plane(D, g, w, ok, x, y, z, core_uv, base, valid, positions, acc);
        prev_ok = ok;
        px = x;
        py = y;
        pz = z;
    }
    flush_stats(stats, q.gi, acc);
}

__global__ void invert_newton_kernel(NewtonGeom G, const double *__restrict__ t,
                                     const double *__restrict__ gs, int64_t n, double tol,
                                     int max_iter, double max_step, double z_floor,
                                     double *__restrict__ pos, uint8_t *__restrict__ ok,
                                     int64_t *__restrict__ iters) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double gz = gs[3 * i + 2] > z_floor ? gs[3 * i + 2] : z_floor;
    double x = gs[3 * i], y = gs[3 * i + 1], z = gz;
    int it = 0, st = 0;
    while (st == 0 && it < max_iter) {
        ++it;
        st = newton_iteration(G, t[3 * i], t[3 * i + 1], t[3 * i + 2], x, y, z, tol,
                              max_step * max_step, max_step, z_floor);
    }
    const bool good = st == 1;
    iters[i] = it;
    ok[i] = good;
    pos[3 * i] = good ? x : gs[3 * i];
    pos[3 * i + 1] = good ? y : gs[3 * i + 1];
    pos[3 * i + 2] = good ? z : gz;
}

}  // namespace hhsar

using namespace hhsar;

extern "C" int hhsar_leaf_boxes(const double *el_pos, const int64_t *bounds, int64_t n_leaves,
                                double *box, void *stream) {
    HHSAR_REQUIRE(n_leaves > 0 && n_leaves < (1ll << 31), "leaf_boxes: bad leaf count");
    leaf_boxes_kernel<<<(unsigned)n_leaves, PLAN_THREADS, 0, as_stream(stream)>>>(el_pos, bounds, box);
    return check_launch("leaf_boxes_kernel");
}

// offset / col_offset of every grid as exclusive prefix sums of the lattice
// sizes and active-column counts the plan just wrote, totals[0] = points,
// totals[1] = columns (one CTA: a few thousand grids at most).
constexpr int SCAN_THREADS = 1024;
__global__ void __launch_bounds__(SCAN_THREADS)
grid_offsets_kernel(hhsar_grid_desc *__restrict__ grids, int n, int64_t *__restrict__ totals) {
    __shared__ int64_t s_p[SCAN_THREADS / 32], s_c[SCAN_THREADS / 32];
    const int per = (n + SCAN_THREADS - 1) / SCAN_THREADS;
    const int a = min(n, (int)threadIdx.x * per), b = min(n, a + per);
    auto sizes = [&](int i, int64_t &pts, int64_t &cols) {
        const hhsar_grid_desc &D = grids[i];
        pts = (int64_t)D.dims[0] * D.dims[1] * D.dims[2];
        const int64_t su = max(D.act_hi[0] - D.act_lo[0] + 1, 0);
        const int64_t sv = max(D.act_hi[1] - D.act_lo[1] + 1, 0);
        cols = su * sv;
    };
    int64_t p = 0, c = 0;
    for (int i = a; i < b; ++i) {
        int64_t pi, ci;
        sizes(i, pi, ci);
        p += pi;
        c += ci;
    }
    // block-wide exclusive scan of (p, c)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t ip = p, ic = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t tp = __shfl_up_sync(0xffffffffu, ip, o);
        const int64_t tc = __shfl_up_sync(0xffffffffu, ic, o);
        if (lane >= o) {
            ip += tp;
            ic += tc;
        }
    }
    if (lane == 31) {
        s_p[wid] = ip;
        s_c[wid] = ic;
    }
    __syncthreads();
    if (wid == 0) {
        int64_t wp = s_p[lane], wc = s_c[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t tp = __shfl_up_sync(0xffffffffu, wp, o);
            const int64_t tc = __shfl_up_sync(0xffffffffu, wc, o);
            if (lane >= o) {
                wp += tp;
                wc += tc;
            }
        }
        s_p[lane] = wp;
        s_c[lane] = wc;
    }
    __syncthreads();
    int64_t op = ip - p + (wid ? s_p[wid - 1] : 0), oc = ic - c + (wid ? s_c[wid - 1] : 0);
    for (int i = a; i < b; ++i) {
        int64_t pi, ci;
        sizes(i, pi, ci);
        grids[i].offset = op;
        grids[i].col_offset = oc;
        op += pi;
        oc += ci;
    }
    if (threadIdx.x == SCAN_THREADS - 1) {
        totals[0] = op;
        totals[1] = oc;
    }
}

// Delay-bin window [b0, b0 + w) the leaf stage can read (ffbp.leaf_range_gate
// restated; same float64 operations, so the same integers).  A valid leaf
// point p lies on a near-band plane w in [near_lo, near_hi] (finish_plane,
// the march ends at near_hi) where Newton converged to n(p) = origin_n +
// step w within tol.  n = c_nhi sqrt(r^2 - gap) - c_nlo r is increasing in
// the vertex distance sum r (dn/dr >= c_nhi - c_nlo > 0), with inverse
//     r(n) = (c_nlo n + c_nhi sqrt(n^2 + (c_nhi^2 - c_nlo^2) gap)) / (c_nhi^2 - c_nlo^2),
// so r(p) lies in [r(n_lo), r(n_hi)].  The four vertices v_i lie within
// Dc of the element-box centre c, so |p - c| lies within r/4 -+ Dc, and the
// leaf kernel's staging windows |p - c| -+ |e - c| (triangle inequality)
// within r/4 -+ (Dc + hd), hd the half 3-D diagonal of the element box;
// every delay it reads lies inside.  4 bins of pad each side cover the
// kernel's +-2-bin windows, floors and fast-path tests.  (The plan's
// containment boxes give a far looser bound: at config 4 valid leaf points
// span 100 bins, the slack boxes 288.)  One CTA.
__global__ void __launch_bounds__(SCAN_THREADS)
leaf_gate_kernel(const hhsar_grid_desc *__restrict__ leaves, int n, hhsar_geom g, double inv_bin,
                 int64_t n_t, int64_t *__restrict__ gate) {
    __shared__ double s_lo[SCAN_THREADS / 32], s_hi[SCAN_THREADS / 32];
    double dmin = DBL_MAX, dmax = 0.0;
    const double A = xsub(xsq(g.c_nhi), xsq(g.c_nlo));
    for (int i = threadIdx.x; i < n; i += SCAN_THREADS) {
        const hhsar_grid_desc &D = leaves[i];
        const double gap = box_gap_exact(D.ext);
        const double Ag = xmul(A, gap);
        const double n_lo = xsub(xadd(D.origin[2], xmul(g.step, (double)D.near_lo[2])), g.tol);
        const double n_hi = xadd(xadd(D.origin[2], xmul(g.step, (double)D.near_hi[2])), g.tol);
        const double r_lo = xdiv(xadd(xmul(g.c_nlo, n_lo), xmul(g.c_nhi, xsqrt(xadd(xsq(n_lo), Ag)))), A);
        const double r_hi = xdiv(xadd(xmul(g.c_nlo, n_hi), xmul(g.c_nhi, xsqrt(xadd(xsq(n_hi), Ag)))), A);
        const double cx = xmul(0.5, xadd(D.box[0], D.box[3]));
        const double cy = xmul(0.5, xadd(D.box[1], D.box[4]));
        const double cz = xmul(0.5, xadd(D.box[2], D.box[5]));
        const double z2 = xsq(cz);
        double dc = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double vx = D.ext[q >> 1], vy = D.ext[2 + (q & 1)];
            dc = fmax(dc, xsqrt(xadd(xadd(xsq(xsub(cx, vx)), xsq(xsub(cy, vy))), z2)));
        }
        const double hd = xmul(0.5, xsqrt(xadd(xadd(xsq(xsub(D.box[3], D.box[0])),
                                                   xsq(xsub(D.box[4], D.box[1]))),
                                              xsq(xsub(D.box[5], D.box[2])))));
        const double pad = xadd(dc, hd);
        dmin = fmin(dmin, xsub(xmul(0.25, r_lo), pad));
        dmax = fmax(dmax, xadd(xmul(0.25, r_hi), pad));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        s_lo[wid] = dmin;
        s_hi[wid] = dmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < SCAN_THREADS / 32; ++k) {
            dmin = fmin(dmin, s_lo[k]);
            dmax = fmax(dmax, s_hi[k]);
        }
        dmin = dmin > 0.0 ? dmin : 0.0;
        int64_t b0 = (int64_t)floor(xmul(dmin, inv_bin)) - 4;
        b0 = b0 > 0 ? b0 : 0;
        int64_t b1 = (int64_t)ceil(xmul(dmax, inv_bin)) + 5;
        b1 = b1 < n_t ? b1 : n_t;
        int64_t w = (b1 - b0 + 31) / 32 * 32;
        w = w < n_t - b0 ? w : n_t - b0;
        gate[0] = b0;
        gate[1] = w;
    }
}

extern "C" int hhsar_leaf_range_gate(const hhsar_grid_desc *leaves, int64_t n_leaves,
                                     const hhsar_geom *geom, double dt, int64_t n_t, int64_t *gate,
                                     void *stream) {
    HHSAR_REQUIRE(n_leaves > 0 && n_leaves < (1ll << 31) && geom != nullptr && dt > 0.0 && n_t > 0,
                  "leaf_range_gate: bad arguments");
    leaf_gate_kernel<<<1, SCAN_THREADS, 0, as_stream(stream)>>>(
        leaves, (int)n_leaves, *geom, 2.0 / (HHSAR_C_LIGHT * dt), n_t, gate);
    return check_launch("leaf_gate_kernel");
}

extern "C" int hhsar_grid_plan(hhsar_grid_desc *grids, int64_t n_grids, const double *leaf_box,
                               const double *boundary, int64_t n_b, const hhsar_geom *geom,
                               int32_t *status, int64_t *totals, void *stream) {
    HHSAR_REQUIRE(n_grids > 0 && n_grids < (1ll << 31), "grid_plan: bad grid count");
    HHSAR_REQUIRE(n_b > 0 && geom != nullptr, "grid_plan: bad boundary lattice");
    HHSAR_REQUIRE(geom->step > 0.0 && geom->step <= 1.0, "grid_plan: step must lie in (0, 1]");
    HHSAR_REQUIRE(geom->max_iter >= 1 && geom->max_iter <= HHSAR_MAX_NEWTON_ITER,
                  "grid_plan: max_iter must lie in [1, 126]");
    grid_plan_kernel<<<(unsigned)n_grids, PLAN_THREADS, 0, as_stream(stream)>>>(
        grids, leaf_box, boundary, (int)n_b, *geom, status);
    if (totals != nullptr) {
        int rc = check_launch("grid_plan_kernel");
        if (rc) return rc;
        grid_offsets_kernel<<<1, SCAN_THREADS, 0, as_stream(stream)>>>(grids, (int)n_grids,
                                                                        totals);
        return check_launch("grid_offsets_kernel");
    }
    return check_launch("grid_plan_kernel");
}

extern "C" int hhsar_grid_newton(const hhsar_grid_desc *grids, int64_t n_grids, int64_t n_cols,
                                 const int32_t *block_grid, const hhsar_geom *geom,
                                 double *positions, uint8_t *valid, int64_t *stats,
                                 void *stream) {
    HHSAR_REQUIRE(n_grids > 0 && n_cols >= 0 && geom != nullptr, "grid_newton: bad sizes");
    // iteration counts travel in 7 bits next to the ok flag (spec_code), and
    // 0xff (ok at 127 iterations) is the "no continuation" sentinel
    HHSAR_REQUIRE(geom->max_iter >= 1 && geom->max_iter <= HHSAR_MAX_NEWTON_ITER,
                  "grid_newton: max_iter must lie in [1, 126]");
    if (n_cols == 0) return HHSAR_OK;
    cudaStream_t s = as_stream(stream);
    const int per_sm = occupancy((const void *)grid_newton_kernel<false>, NEWTON_THREADS);
    const int per_sm2 = occupancy((const void *)grid_newton_kernel<true>, NEWTON_THREADS);
    // Speculative warm continuations of the heavy planes (SPEC2) pay where
    // the in-order fix-up is the critical path, i.e. small problems (config
    // 2: 39 k columns); on large ones the heavy phase is throughput work
    // competing with the range compression, and they are off.
    const bool spec2 = n_cols <= NEWTON_SPEC2_MAX_COLS;
    const int64_t cap = spec2 ? (n_cols / 8 > 256 ? n_cols / 8 : 256) : 0;  // heavy columns with slots
    // scratch: [0] work counter, [1] heavy-column count, then the heavy list,
    // the column -> grid map, and (SPEC2) the continuation slots
    unsigned long long *counter = nullptr;
    const size_t head = 2 * sizeof(unsigned long long) + 2 * n_cols * sizeof(int32_t);
    const size_t slots = (size_t)cap * HEAVY_MAXP * SPEC_DEPTH;
    if (cudaMallocAsync(&counter, head + slots * (3 * sizeof(double) + 1), s) != cudaSuccess)
        return set_error(HHSAR_ECUDA, "grid_newton: scratch allocation failed");
    cudaMemsetAsync(counter, 0, 2 * sizeof(unsigned long long), s);
    int32_t *heavy = reinterpret_cast<int32_t *>(counter + 2);
    int32_t *col_grid = heavy + n_cols;
    double *spec2_pos = spec2 ? reinterpret_cast<double *>(col_grid + n_cols) : nullptr;
    uint8_t *spec2_code = spec2 ? reinterpret_cast<uint8_t *>(spec2_pos + 3 * slots) : nullptr;
    if (spec2) cudaMemsetAsync(spec2_code, 0xff, slots, s);  // 0xff = no continuation
    grid_newton_heavy_list_kernel<<<(unsigned)((n_cols + 255) / 256), 256, 0, s>>>(
        grids, (int)n_grids, n_cols, block_grid, *geom, heavy, counter + 1, col_grid);
    // every task is short (a heavy plane or a light column), so full occupancy.
    // 1. heavy planes; 2. the light columns on `s` while the latency-bound
    // in-order fix-up of the heavy columns runs beside them on a side stream
    const int64_t blocks = (int64_t)sm_count() * per_sm;
    if (spec2)
        grid_newton_kernel<true><<<(unsigned)(sm_count() * per_sm2), NEWTON_THREADS, 0, s>>>(
            grids, (int)n_grids, n_cols, block_grid, *geom, positions, valid, stats, counter,
            heavy, counter + 1, 0, col_grid, spec2_pos, spec2_code, cap);
    else
        grid_newton_kernel<false><<<(unsigned)blocks, NEWTON_THREADS, 0, s>>>(
            grids, (int)n_grids, n_cols, block_grid, *geom, positions, valid, stats, counter,
            heavy, counter + 1, 0, col_grid, nullptr, nullptr, 0);
    // the fix-up runs on the device's high-priority side stream (it must not
    // queue behind range-compression CTAs); fork/join events are per call
    cudaStream_t side = side_stream();
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    if (side == nullptr || cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&join_ev, cudaEventDisableTiming) != cudaSuccess) {
        if (fork_ev) cudaEventDestroy(fork_ev);
        side = s;  // no side stream: run the fix-up in order on the caller's stream
        fork_ev = join_ev = nullptr;
    }
    if (fork_ev) {
        cudaEventRecord(fork_ev, s);
        cudaStreamWaitEvent(side, fork_ev, 0);
    }
    grid_newton_fixup_kernel<<<(unsigned)((n_cols + NEWTON_THREADS - 1) / NEWTON_THREADS),
                               NEWTON_THREADS, 0, side>>>(grids, (int)n_grids, block_grid, *geom,
                                                          positions, valid, stats, heavy,
                                                          counter + 1, col_grid, spec2_pos,
                                                          spec2_code, cap);
    if (join_ev) cudaEventRecord(join_ev, side);
    cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s);  // work counter for phase 1
    grid_newton_kernel<false><<<(unsigned)blocks, NEWTON_THREADS, 0, s>>>(
        grids, (int)n_grids, n_cols, block_grid, *geom, positions, valid, stats, counter, heavy,
        counter + 1, 1, col_grid, nullptr, nullptr, 0);
    if (join_ev) {
        cudaStreamWaitEvent(s, join_ev, 0);
        cudaEventDestroy(fork_ev);  // released once the recorded work completes
        cudaEventDestroy(join_ev);
    }
    cudaFreeAsync(counter, s);
    return check_launch("grid_newton_kernel / grid_newton_fixup_kernel");
}

extern "C" int hhsar_invert_newton(const double *ext4, double k_min, double k_max,
                                   const double *targets, const double *guesses, int64_t n,
                                   double tol, int max_iter, double max_step, double z_floor,
                                   double *pos, uint8_t *ok, int64_t *iters, void *stream) {
    HHSAR_REQUIRE(n >= 0 && max_iter >= 1, "invert_newton: bad arguments");
    if (n == 0) return HHSAR_OK;
    NewtonGeom G;
    for (int k = 0; k < 4; ++k) G.ext[k] = ext4[k];
    G.gap = 4.0 * (ext4[1] - ext4[0]) * (ext4[1] - ext4[0]) +
            4.0 * (ext4[3] - ext4[2]) * (ext4[3] - ext4[2]);
    const double pi = 3.141592653589793;
    G.c_uv = k_max / pi;
    G.c_nhi = k_max / (4.0 * pi);
    G.c_nlo = k_min / (4.0 * pi);
    invert_newton_kernel<<<(unsigned)((n + 127) / 128), 128, 0, as_stream(stream)>>>(
        G, targets, guesses, n, tol, max_iter, max_step > 0 ? max_step : 0.0, z_floor, pos, ok,
        iters);
    return check_launch("invert_newton_kernel");
}
