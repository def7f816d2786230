"""CPU checks of the algebra behind two kernels, restated in numpy float64
(no GPU): the one-exchange split range compression (range_sim.cu,
range_compress_split_kernel) and the z-series Cartesian landing
(leaf_merge.cu, merge_cartesian_series_kernel).  The GPU tests compare the
kernels with the oracle; these pin the decompositions themselves."""

import numpy as np
import pytest


def _split_window(x, n_t, b0, w):
    """range_compress_split_kernel's decomposition for one row: n = 64 n1 +
    n2, k = k1 + KC k2 (KC = n_t / 64); stage A per column n2 as four
    (KC/4)-point DFTs (k1 = 4 q + r); stage B per thread t: bins
    kb + 64 o (kb = b0 + t), n2 = 16 a + b, one S-point combination per b
    (S = n_t / 1024) feeding a 16-term Horner chain in z = W^k."""
    kc = n_t // 64
    nl = x.size // 64
    W = lambda m, k: np.exp(2j * np.pi * k / m)  # noqa: E731
    xs = x.reshape(nl, 64)  # [n1][n2]
    cols = np.zeros((kc, 64), complex)  # [k1][n2]
    for r in range(4):
        y = xs * W(kc, np.arange(nl) * r)[:, None]
        for q in range(kc // 4):
            cols[4 * q + r] = (y * W(kc // 4, np.arange(nl) * q)[:, None]).sum(axis=0)
    s = n_t // 1024
    out = np.zeros(w, complex)
    for t in range(64):
        kb = b0 + t
        col = cols[kb % kc]
        tau = [W(n_t, 16 * a * kb) for a in range(4)]
        o = 0
        while t + 64 * o < w:
            k = kb + 64 * o
            z = W(n_t, k)
            acc = 0j
            for b in range(15, -1, -1):
                v = [tau[a] * col[16 * a + b] for a in range(4)]
                zb = sum(v[a] * W(s, a * (o % s)) for a in range(4))
                acc = acc * z + zb
            out[t + 64 * o] = acc
            o += 1
    return out


@pytest.mark.parametrize("n_f,n_t,b0,w", [(1024, 4096, 49, 288), (512, 4096, 3000, 400),
                                          (512, 2048, 0, 352), (256, 2048, 1600, 448),
                                          (1024, 4096, 4095, 1)])
def test_split_range_compression_algebra(n_f, n_t, b0, w):
    rng = np.random.default_rng(n_f + b0)
    x = rng.standard_normal(n_f) + 1j * rng.standard_normal(n_f)
    pad = np.zeros(n_t, complex)
    pad[:n_f] = x
    want = (np.fft.ifft(pad) * n_t)[b0:b0 + w]  # unnormalised inverse DFT
    got = _split_window(x, n_t, b0, w)
    assert np.max(np.abs(got - want)) <= 1e-9 * np.max(np.abs(want))


def _d_series(s, z):
    """Taylor coefficients d^(k)(z)/k!, k <= 4, of d = sqrt(s + z^2) (the
    kernel's y = 1/d forms)."""
    a = s + z * z
    y = 1.0 / np.sqrt(a)
    return np.array([a * y, z * y, 0.5 * s * y ** 3, -0.5 * s * z * y ** 5,
                     s * (4 * z * z - s) * y ** 7 / 8])


def _sqrt_series(U):
    S = np.zeros(5)
    S[0] = np.sqrt(U[0])
    hw = 0.5 / S[0]
    S[1] = U[1] * hw
    S[2] = (U[2] - S[1] ** 2) * hw
    S[3] = (U[3] - 2 * S[1] * S[2]) * hw
    S[4] = (U[4] - 2 * S[1] * S[3] - S[2] ** 2) * hw
    return S


def _recip_series(D):
    C = np.zeros(5)
    C[0] = 1.0 / D[0]
    for m in range(1, 5):
        C[m] = -sum(D[q] * C[m - q] for q in range(1, m + 1)) * C[0]
    return C


@pytest.mark.parametrize("zmin,zmax,nz,zq", [(0.3, 0.4, 256, 8), (0.20475, 0.39525, 128, 8),
                                             (0.2035, 0.2965, 32, 4)])
def test_landing_z_series_algebra(zmin, zmax, nz, zq):
    """The landing's per-block quartic series of r = sum of the four corner
    distances, sq = sqrt(r^2 - gap), the phase 0.25 (k_max sq + k_min r)
    and 1 / (d_a + d_b) against direct float64 evaluation over the block
    (configs 4 / 3 / 0 geometry: ZQ = 8 / 8 / 4 as the launcher picks)."""
    sz = (zmax - zmin) / (nz - 1)
    assert (zq - 1) / 2 * sz <= 0.06 * zmin  # the launcher's rule holds here
    rng = np.random.default_rng(nz + zq)
    k_min, k_max = 1571.9, 1781.5
    worst_phase = worst_r = worst_u = 0.0
    for _ in range(300):
        x, y = rng.uniform(-0.16, 0.16, 2)
        e = np.sort(rng.uniform(-0.21, 0.14, 2))
        f = np.sort(rng.uniform(-0.21, 0.13, 2))
        gap = 4 * (e[1] - e[0]) ** 2 + 4 * (f[1] - f[0]) ** 2
        kblk = rng.integers(0, nz // zq)
        zc = zmin + sz * (kblk * zq + 0.5 * (zq - 1))
        ss = [(x - e[i]) ** 2 + (y - f[j]) ** 2 for i in (0, 1) for j in (0, 1)]
        R = sum(_d_series(s, zc) for s in ss)
        U = np.array([R[0] ** 2 - gap, 2 * R[0] * R[1], R[1] ** 2 + 2 * R[0] * R[2],
                      2 * R[0] * R[3] + 2 * R[1] * R[2],
                      2 * R[0] * R[4] + 2 * R[1] * R[3] + R[2] ** 2])
        S = _sqrt_series(U)
        P = 0.25 * (k_max * S + k_min * R)
        dy0 = y - f[0] if y < f[0] else (y - f[1] if y > f[1] else 0.0)
        qa, qb = (x - e[0]) ** 2 + dy0 ** 2, (x - e[1]) ** 2 + dy0 ** 2
        Cr = _recip_series(_d_series(qa, zc) + _d_series(qb, zc))
        for j in range(zq):
            t = (j - 0.5 * (zq - 1)) * sz
            z = zc + t
            r = sum(np.sqrt(s + z * z) for s in ss)
            sq = np.sqrt(r * r - gap)
            phase = 0.25 * (k_max * sq + k_min * r)
            poly = lambda c: sum(c[m] * t ** m for m in range(5))  # noqa: E731
            worst_phase = max(worst_phase, abs(poly(P) - phase))
            worst_r = max(worst_r, abs(poly(R) - r))
            inv = 1.0 / (np.sqrt(qa + z * z) + np.sqrt(qb + z * z))
            worst_u = max(worst_u, abs(poly(Cr) - inv) / inv)
    assert worst_phase < 1e-5, worst_phase  # rad (the float32 terms add ~1e-6)
    assert worst_r < 1e-8, worst_r          # m
    assert worst_u < 1e-7, worst_u          # relative, as the float32 u/v form
