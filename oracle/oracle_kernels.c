/*
 * TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's three hot
 * loops (/root/reference/pkg/src/hhsar/_kernels.py).  Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline leg may load this
 * library, and only as the checker / the timed CPU baseline.  The product
 * path (paper_2506_23568_b200) never links or calls it.
 *
 * Arithmetic is IEEE float64 (the reference uses Numba fastmath float64; the
 * two agree to ~1e-14 relative, see tests/test_oracle_golden.py).
 * Parallelism is OpenMP over points, like the reference's prange.
 */
#include <math.h>
#include <stdint.h>
#include <omp.h>

#define C_LIGHT 299792458.0

static void set_threads(int threads) {
    if (threads > 0) omp_set_num_threads(threads);
}

int oracle_max_threads(void) { return omp_get_max_threads(); }

/* _kernels.py:44-75 -- per point, sum over elements of the linearly
 * interpolated envelope times the carrier exp(j k_ref c tau).  Delays with
 * x outside [0, n_t-1] are skipped and counted. */
void oracle_bp_gather(const double *pts, int64_t n, const double *el, int64_t m,
                      const double *env, int64_t n_t, double t0, double dt,
                      double k_ref, double *out, int64_t *oow, int threads) {
    set_threads(threads);
    const double kc = k_ref * C_LIGHT;
    #pragma omp parallel for schedule(dynamic, 64)
    for (int64_t p = 0; p < n; ++p) {
        const double px = pts[3 * p], py = pts[3 * p + 1], pz = pts[3 * p + 2];
        double ar = 0.0, ai = 0.0;
        int64_t bad = 0;
        for (int64_t e = 0; e < m; ++e) {
            const double dx = px - el[3 * e], dy = py - el[3 * e + 1],
                         dz = pz - el[3 * e + 2];
            const double tau = 2.0 * sqrt(dx * dx + dy * dy + dz * dz) / C_LIGHT;
            const double x = (tau - t0) / dt;
            if (x < 0.0 || x > (double)(n_t - 1)) { ++bad; continue; }
            int64_t i = (int64_t)x;
            if (i > n_t - 2) i = n_t - 2;
            const double f = x - (double)i;
            const double *row = env + 2 * (e * n_t + i);
            const double vr = row[0] * (1.0 - f) + row[2] * f;
            const double vi = row[1] * (1.0 - f) + row[3] * f;
            const double ph = kc * tau, c = cos(ph), s = sin(ph);
            ar += vr * c - vi * s;
            ai += vr * s + vi * c;
        }
        out[2 * p] = ar;
        out[2 * p + 1] = ai;
        oow[p] = bad;
    }
}

/* simulator.py:41-69 -- first-order Born cube
 * s[e][f] = sum_q refl_q exp(-2j k_f |el_e - pos_q|), float64. */
void oracle_simulate(const double *el, int64_t n_el, const double *pos, const double *refl,
                     int64_t n_s, const double *k, int64_t n_f, double *out, int threads) {
    set_threads(threads);
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n_el; ++e) {
        double *row = out + 2 * e * n_f;
        for (int64_t f = 0; f < n_f; ++f) { row[2 * f] = 0.0; row[2 * f + 1] = 0.0; }
        for (int64_t q = 0; q < n_s; ++q) {
            const double dx = el[3 * e] - pos[3 * q], dy = el[3 * e + 1] - pos[3 * q + 1],
                         dz = el[3 * e + 2] - pos[3 * q + 2];
            const double d = sqrt(dx * dx + dy * dy + dz * dz);
            const double rr = refl[2 * q], ri = refl[2 * q + 1];
            for (int64_t f = 0; f < n_f; ++f) {
                const double ph = -2.0 * k[f] * d, c = cos(ph), s = sin(ph);
                row[2 * f] += rr * c - ri * s;
                row[2 * f + 1] += rr * s + ri * c;
            }
        }
    }
}

static void keys4(double f, double w[4]) { /* _kernels.py:192-200, a = -1/2 */
    w[0] = ((-0.5 * f + 1.0) * f - 0.5) * f;
    w[1] = (1.5 * f - 2.5) * f * f + 1.0;
    w[2] = ((-1.5 * f + 2.0) * f + 0.5) * f;
    w[3] = (0.5 * f - 0.5) * f * f;
}

/* _kernels.py:117-189 -- separable trilinear (cubic=0) or Keys-cubic
 * (cubic=1) interpolation of a [nu][nv][nn] complex lattice at fractional
 * lattice coordinates; out-of-hull points return 0 with ok = 0. */
void oracle_interp(const double *vals, int64_t nu, int64_t nv, int64_t nn,
                   const double *coords, int64_t n, int cubic, double *out,
                   uint8_t *ok, int threads) {
    set_threads(threads);
    #pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < n; ++p) {
        const double cu = coords[3 * p], cv = coords[3 * p + 1], cn = coords[3 * p + 2];
        out[2 * p] = 0.0;
        out[2 * p + 1] = 0.0;
        ok[p] = 0;
        double ar = 0.0, ai = 0.0;
        if (!cubic) {
            if (cu < 0.0 || cu > (double)(nu - 1) || cv < 0.0 || cv > (double)(nv - 1) ||
                cn < 0.0 || cn > (double)(nn - 1)) continue;
            int64_t iu = (int64_t)cu, iv = (int64_t)cv, iw = (int64_t)cn;
            if (iu > nu - 2) iu = nu - 2;
            if (iv > nv - 2) iv = nv - 2;
            if (iw > nn - 2) iw = nn - 2;
            const double fu = cu - iu, fv = cv - iv, fn = cn - iw;
            for (int a = 0; a < 2; ++a) {
                const double wa = a ? fu : 1.0 - fu;
                for (int b = 0; b < 2; ++b) {
                    const double wb = b ? fv : 1.0 - fv;
                    for (int c = 0; c < 2; ++c) {
                        const double wc = c ? fn : 1.0 - fn;
                        const double w = wa * wb * wc;
                        const double *v = vals + 2 * (((iu + a) * nv + iv + b) * nn + iw + c);
                        ar += v[0] * w;
                        ai += v[1] * w;
                    }
                }
            }
        } else {
            if (cu < 1.0 || cu > (double)(nu - 2) || cv < 1.0 || cv > (double)(nv - 2) ||
                cn < 1.0 || cn > (double)(nn - 2)) continue;
            int64_t iu = (int64_t)cu, iv = (int64_t)cv, iw = (int64_t)cn;
            if (iu > nu - 3) iu = nu - 3;
            if (iv > nv - 3) iv = nv - 3;
            if (iw > nn - 3) iw = nn - 3;
            double wu[4], wv[4], wn[4];
            keys4(cu - iu, wu);
            keys4(cv - iv, wv);
            keys4(cn - iw, wn);
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b)
                    for (int c = 0; c < 4; ++c) {
                        const double w = wu[a] * wv[b] * wn[c];
                        const double *v = vals + 2 * (((iu - 1 + a) * nv + iv - 1 + b) * nn + iw - 1 + c);
                        ar += v[0] * w;
                        ai += v[1] * w;
                    }
        }
        out[2 * p] = ar;
        out[2 * p + 1] = ai;
        ok[p] = 1;
    }
}

/* _kernels.py:255-351 -- damped Newton inversion of the (u, v, n) map with
 * the analytic Jacobian and a Cramer solve; trust radius max_step (<= 0
 * disables it), z floored to z_floor.  Failed points return their
 * (z-floored) guess with ok = 0. */
void oracle_newton(double x_min, double x_max, double y_min, double y_max,
                   double k_min, double k_max, const double *targets,
                   const double *guesses, int64_t n, double tol, int max_iter,
                   double max_step, double z_floor, double *pos, uint8_t *ok,
                   int64_t *iters, int threads) {
    set_threads(threads);
    const double gap = 4.0 * (x_max - x_min) * (x_max - x_min)
                     + 4.0 * (y_max - y_min) * (y_max - y_min);
    const double pi = M_PI;
    const double cu = k_max / pi, cn_hi = k_max / (4.0 * pi), cn_lo = k_min / (4.0 * pi);
    #pragma omp parallel for schedule(dynamic, 32)
    for (int64_t i = 0; i < n; ++i) {
        const double gz = guesses[3 * i + 2] > z_floor ? guesses[3 * i + 2] : z_floor;
        double x = guesses[3 * i], y = guesses[3 * i + 1], z = gz;
        const double tu = targets[3 * i], tv = targets[3 * i + 1], tn = targets[3 * i + 2];
        int good = 0, it = 0;
        for (it = 1; it <= max_iter; ++it) {
            const double x0 = fmin(fmax(x, x_min), x_max);
            const double y0 = fmin(fmax(y, y_min), y_max);
            const double z2 = z * z;
            const double ax = x - x_min, bx = x - x_max, ay = y - y_min, by = y - y_max;
            const double du1 = sqrt(ax * ax + (y - y0) * (y - y0) + z2);
            const double du2 = sqrt(bx * bx + (y - y0) * (y - y0) + z2);
            const double dv1 = sqrt((x - x0) * (x - x0) + ay * ay + z2);
            const double dv2 = sqrt((x - x0) * (x - x0) + by * by + z2);
            const double e1 = sqrt(ax * ax + ay * ay + z2);
            const double e2 = sqrt(ax * ax + by * by + z2);
            const double e3 = sqrt(bx * bx + ay * ay + z2);
            const double e4 = sqrt(bx * bx + by * by + z2);
            const double r = e1 + e2 + e3 + e4;
            const double rad = r * r - gap;
            if (rad <= 0.0 || fmin(fmin(du1, du2), fmin(dv1, dv2)) == 0.0 ||
                fmin(fmin(e1, e2), fmin(e3, e4)) == 0.0) break;
            const double sq = sqrt(rad);
            const double ru = cu * (du1 - du2) - tu;
            const double rv = cu * (dv1 - dv2) - tv;
            const double rn = cn_hi * sq - cn_lo * r - tn;
            if (fmax(fabs(ru), fmax(fabs(rv), fabs(rn))) <= tol) { good = 1; break; }
            const double ja = cu * (ax / du1 - bx / du2);
            const double jb = cu * ((y - y0) / du1 - (y - y0) / du2);
            const double jc = cu * (z / du1 - z / du2);
            const double jd = cu * ((x - x0) / dv1 - (x - x0) / dv2);
            const double je = cu * (ay / dv1 - by / dv2);
            const double jf = cu * (z / dv1 - z / dv2);
            const double fac = cn_hi * (r / sq) - cn_lo;
            const double jg = fac * (ax / e1 + ax / e2 + bx / e3 + bx / e4);
            const double jh = fac * (ay / e1 + by / e2 + ay / e3 + by / e4);
            const double ji = fac * (z / e1 + z / e2 + z / e3 + z / e4);
            const double m0 = je * ji - jf * jh, m1 = jd * ji - jf * jg, m2 = jd * jh - je * jg;
            const double det = ja * m0 - jb * m1 + jc * m2;
            if (fabs(det) < 1e-30) break;
            double sx = (ru * m0 - jb * (rv * ji - jf * rn) + jc * (rv * jh - je * rn)) / det;
            double sy = (ja * (rv * ji - jf * rn) - ru * m1 + jc * (jd * rn - rv * jg)) / det;
            double sz = (ja * (je * rn - rv * jh) - jb * (jd * rn - rv * jg) + ru * m2) / det;
            if (max_step > 0.0) {
                const double sn = sqrt(sx * sx + sy * sy + sz * sz);
                if (sn > max_step) {
                    const double sc = max_step / sn;
                    sx *= sc; sy *= sc; sz *= sc;
                }
            }
            x -= sx; y -= sy; z -= sz;
            if (z < z_floor) z = z_floor;
        }
        if (it > max_iter) it = max_iter;
        iters[i] = it;
        if (good) {
            pos[3 * i] = x; pos[3 * i + 1] = y; pos[3 * i + 2] = z; ok[i] = 1;
        } else {
            pos[3 * i] = guesses[3 * i]; pos[3 * i + 1] = guesses[3 * i + 1];
            pos[3 * i + 2] = gz; ok[i] = 0;
        }
    }
}
