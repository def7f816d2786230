"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference hot path.

Each function cites the reference code it restates (paths relative to
/root/reference/pkg/src/hhsar/).  The three inner loops run in the OpenMP C
library ``oracle_kernels.c`` (built on demand with gcc into oracle/_build/);
everything else is float64 numpy.  Inputs are duck-typed: the reference's
objects, the product package's objects, or anything with the same fields.

Pinned against the reference's own outputs: tests/golden/*.npz are written by
tests/golden/make_golden.py, which imports the reference in the build
container; tests/test_oracle_golden.py checks this module against them.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

__all__ = [
    "C_LIGHT", "GRID_PAD", "OracleError", "OracleDomainError", "OracleConfigError",
    "Profiles", "Grid", "Sub", "range_compress", "region_grid", "check_delay_window",
    "bp_gather", "backproject", "bpa_reconstruct", "extents_of", "sdc_phase",
    "llt_forward", "invert_newton", "interpolate", "build_grid", "level1",
    "merge_onto_points", "merge_children", "hhffbpa_reconstruct",
    "default_grid_dims", "leaf_bounds", "tree_levels", "threads", "simulate",
    "Plan", "plan_grid", "grid_levels",
]

C_LIGHT = 299792458.0
GRID_PAD = 2  # ffbp.py:32
TWO_PI = 2.0 * np.pi


class OracleError(Exception):
    pass


class OracleDomainError(OracleError):
    """Reference NumericDomainError."""


class OracleConfigError(OracleError):
    """Reference ConfigError."""


# --------------------------------------------------------------------------
# native loops
# --------------------------------------------------------------------------

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"
_lib = None


def build_library(force: bool = False) -> Path:
    """Compile oracle_kernels.c with gcc -O2 -fopenmp (no fast-math)."""
    src = _HERE / "oracle_kernels.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        _LIB_PATH.parent.mkdir(exist_ok=True)
        tmp = _LIB_PATH.with_suffix(f".{os.getpid()}.tmp")
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared",
                               "-std=c99", "-D_DEFAULT_SOURCE", str(src),
                               "-o", str(tmp), "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _native():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(str(build_library()))
        P, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        lib.oracle_bp_gather.argtypes = [P, I64, P, I64, P, I64, D, D, D, P, P, I]
        lib.oracle_interp.argtypes = [P, I64, I64, I64, P, I64, I, P, P, I]
        lib.oracle_newton.argtypes = [D, D, D, D, D, D, P, P, I64, D, I, D, D, P, P, P, I]
        lib.oracle_simulate.argtypes = [P, I64, P, P, I64, P, I64, P, I]
        lib.oracle_max_threads.restype = I
        _lib = lib
    return _lib


_THREADS = int(os.environ.get("ORACLE_THREADS", "0"))


def threads() -> int:
    """Worker threads the C loops use (all host cores unless ORACLE_THREADS)."""
    return _THREADS if _THREADS > 0 else _native().oracle_max_threads()


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def bp_gather(points, el_pos, envelopes, t0, dt, k_ref):
    """_kernels.py:98-110 -> (values complex128 [n], oow int64 [n])."""
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    el = np.ascontiguousarray(el_pos, dtype=np.float64).reshape(-1, 3)
    env = np.ascontiguousarray(envelopes, dtype=np.complex128)
    out = np.zeros(pts.shape[0], dtype=np.complex128)
    oow = np.zeros(pts.shape[0], dtype=np.int64)
    if pts.shape[0] and el.shape[0]:
        _native().oracle_bp_gather(_ptr(pts), pts.shape[0], _ptr(el), el.shape[0],
                                   _ptr(env), env.shape[1], float(t0), float(dt),
                                   float(k_ref), _ptr(out), _ptr(oow), _THREADS)
    return out, oow


def simulate(elements, positions, refl, k_samples):
    """simulator.py:41-69 Born cube, complex128 [N_el, n_f]."""
    el = np.ascontiguousarray(elements, dtype=np.float64).reshape(-1, 3)
    pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    r = np.ascontiguousarray(np.asarray(refl, dtype=np.complex128))
    k = np.ascontiguousarray(k_samples, dtype=np.float64)
    out = np.zeros((el.shape[0], k.size), dtype=np.complex128)
    _native().oracle_simulate(_ptr(el), el.shape[0], _ptr(pos), _ptr(r), pos.shape[0],
                              _ptr(k), k.size, _ptr(out), _THREADS)
    return out


def interpolate(values, coords, kernel="linear"):
    """_kernels.py:354-378 -> (values complex128 [n], ok bool [n])."""
    if kernel not in ("linear", "cubic"):
        raise OracleConfigError(f"unknown interpolation kernel '{kernel}'")
    vals = np.ascontiguousarray(values, dtype=np.complex128)
    c = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(c.shape[0], dtype=np.complex128)
    ok = np.zeros(c.shape[0], dtype=np.uint8)
    if c.shape[0]:
        nu, nv, nn = vals.shape
        _native().oracle_interp(_ptr(vals), nu, nv, nn, _ptr(c), c.shape[0],
                                int(kernel == "cubic"), _ptr(out), _ptr(ok), _THREADS)
    return out, ok.astype(bool)


def invert_newton(ext, targets, guesses, k_min, k_max, tol=1e-9, max_iter=50,
                  max_step=0.0, z_floor=1e-4):
    """_kernels.py:255-351 via spectrum.py:363-370 -> (pos, ok, iters)."""
    t = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 3)
    g = np.ascontiguousarray(guesses, dtype=np.float64).reshape(-1, 3)
    n = t.shape[0]
    pos = np.empty((n, 3))
    ok = np.zeros(n, dtype=np.uint8)
    it = np.zeros(n, dtype=np.int64)
    if n:
        _native().oracle_newton(ext[0], ext[1], ext[2], ext[3], k_min, k_max,
                                _ptr(t), _ptr(g), n, float(tol), int(max_iter),
                                float(max_step or 0.0), float(z_floor), _ptr(pos),
                                _ptr(ok), _ptr(it), _THREADS)
    return pos, ok.astype(bool), it


# --------------------------------------------------------------------------
# range compression and the direct BPA
# --------------------------------------------------------------------------

@dataclass
class Profiles:
    """RangeProfileSet (rangecomp.py:24-58): envelopes[N_el, n_t]."""
    envelopes: np.ndarray
    t0: float
    dt: float
    k_ref: float
    elements: np.ndarray

    @property
    def window(self):
        return (self.t0, self.t0 + (self.envelopes.shape[1] - 1) * self.dt)


def _band(freqs):
    k_min = 2.0 * np.pi * freqs.f_min / C_LIGHT
    k_max = 2.0 * np.pi * freqs.f_max / C_LIGHT
    return k_min, k_max


def range_compress(cube, upsample=8) -> Profiles:
    """rangecomp.py:61-101: zero-padded unnormalised IDFT, then demodulation
    from the band start to the band centre carrier."""
    if int(upsample) != upsample or upsample < 1:
        raise OracleConfigError("upsample factor must be an integer >= 1")
    f = cube.freqs
    k_min, k_max = _band(f)
    n_f = int(f.count)
    n_t = int(upsample) * n_f
    dt = 2.0 * np.pi / (n_t * ((k_max - k_min) / (n_f - 1)) * C_LIGHT)
    k_ref = 0.5 * (k_min + k_max)
    spec = np.zeros((cube.values.shape[0], n_t), dtype=np.complex128)
    spec[:, :n_f] = cube.values
    prof = np.fft.ifft(spec, axis=1) * n_t
    demod = np.exp(1j * (k_min - k_ref) * C_LIGHT * (dt * np.arange(n_t)))
    return Profiles(envelopes=prof * demod, t0=0.0, dt=dt, k_ref=k_ref,
                    elements=np.asarray(cube.aperture.elements, dtype=float))


def _bounds(region):
    return np.array([[region.x_min, region.x_max], [region.y_min, region.y_max],
                     [region.z_min, region.z_max]], dtype=float)


def region_grid(region, dims):
    """bpa.py:73-83: edge-to-edge uniform grid; single-sample axes sit at
    the centre with step = extent."""
    d = np.array([int(v) for v in dims])
    if d.shape != (3,) or np.any(d < 1):
        raise OracleConfigError("grid dims must be three integers >= 1")
    b = _bounds(region)
    lo, hi = b[:, 0], b[:, 1]
    origin = np.where(d > 1, lo, (lo + hi) / 2)
    step = np.where(d > 1, (hi - lo) / np.maximum(d - 1, 1), hi - lo)
    return origin, step


def default_grid_dims(region, freqs):
    """spectrum.py:534-545: resolution-limit grid of the band."""
    k_max = _band(freqs)[1]
    rates = (np.pi / (2.0 * k_max), np.pi / (2.0 * k_max), np.pi / k_max)
    ext = _bounds(region) @ np.array([-1.0, 1.0])
    return tuple(int(round(e / r)) + 1 for e, r in zip(ext, rates))


def check_delay_window(prof: Profiles, region):
    """bpa.py:130-141: farthest region corner vs the profile window."""
    b = _bounds(region)
    corners = np.array([(x, y, z) for x in b[0] for y in b[1] for z in b[2]])
    d = np.sqrt(((corners[None] - prof.elements[:, None]) ** 2).sum(-1))
    tau = 2.0 * d.max() / C_LIGHT
    lo, hi = prof.window
    if tau > hi or 0.0 < lo:
        raise OracleDomainError("max round-trip delay exceeds the profile window")


def backproject(prof: Profiles, sel, points):
    """bpa.py:97-127 with _element_block (bpa.py:86-94)."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    if isinstance(sel, tuple):
        sel = slice(*sel)
    el, env = prof.elements[sel], prof.envelopes[sel]
    if el.shape[0] == 0:
        return np.zeros(pts.shape[0], dtype=complex)
    out, oow = bp_gather(pts, el, env, prof.t0, prof.dt, prof.k_ref)
    if oow.sum():
        raise OracleDomainError(f"{int(oow.sum())} point-element delays fell "
                                "outside the profile window")
    return out


def _mesh(origin, step, dims):
    axes = [origin[a] + step[a] * np.arange(dims[a]) for a in range(3)]
    g = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel() for m in g], axis=-1)


def _validate(cube, region):
    if region.z_min <= float(np.asarray(cube.aperture.elements)[:, 2].max()):
        raise OracleConfigError("region must sit in front of the aperture")


def bpa_reconstruct(cube, region, dims=None, upsample=8, profiles=None):
    """bpa.py:144-176 -> (values[nx,ny,nz] complex128, origin, step, provenance).

    ``profiles`` lets a caller pass a precomputed range compression (the
    BASELINE.md plan times the path with and without range compression).
    """
    _validate(cube, region)
    dims = tuple(int(d) for d in (dims or default_grid_dims(region, cube.freqs)))
    origin, step = region_grid(region, dims)
    prof = profiles if profiles is not None else range_compress(cube, upsample)
    check_delay_window(prof, region)
    vals = backproject(prof, slice(None), _mesh(origin, step, dims))
    return vals.reshape(dims), origin, step, {"algorithm": "bpa", "upsample": upsample,
                                              "dims": list(dims)}


# --------------------------------------------------------------------------
# analytic spectrum geometry (spectrum.py)
# --------------------------------------------------------------------------

def extents_of(elements, start=None, stop=None):
    """SubarrayExtents.from_aperture (spectrum.py:46-54): lateral bbox."""
    e = np.asarray(elements)[start:stop]
    return (float(e[:, 0].min()), float(e[:, 0].max()),
            float(e[:, 1].min()), float(e[:, 1].max()))


def _corner_sum(ext, p):
    # spectrum.py:124-139: ((daa + dab) + dba) + dbb with z' = 0 vertices
    p = np.asarray(p, dtype=float)
    z2 = p[..., 2] ** 2
    xa, xb = (p[..., 0] - ext[0]) ** 2, (p[..., 0] - ext[1]) ** 2
    ya, yb = (p[..., 1] - ext[2]) ** 2, (p[..., 1] - ext[3]) ** 2
    return ((np.sqrt(xa + ya + z2) + np.sqrt(xa + yb + z2))
            + np.sqrt(xb + ya + z2)) + np.sqrt(xb + yb + z2)


def _gap(ext):
    return 4.0 * (ext[1] - ext[0]) ** 2 + 4.0 * (ext[3] - ext[2]) ** 2


def sdc_phase(ext, p, k_min, k_max):
    """spectrum.py:229-240 (Eq. 30): 1/4 k_max sqrt(rad) + 1/4 k_min r."""
    r = _corner_sum(ext, p)
    rad = r * r - _gap(ext)
    if np.any(rad <= _gap(ext) * 1e-12):
        raise OracleDomainError("downconversion phase undefined")
    return 0.25 * k_max * np.sqrt(rad) + 0.25 * k_min * r


def llt_forward(ext, p, k_min, k_max):
    """spectrum.py:243-275 (Eq. 37): compressed (u, v, n) coordinates."""
    p = np.asarray(p, dtype=float)
    x, y, z = p[..., 0], p[..., 1], p[..., 2]
    z2 = z ** 2
    y0 = np.clip(y, ext[2], ext[3])
    x0 = np.clip(x, ext[0], ext[1])
    dy0 = (y - y0) ** 2
    u = (k_max / np.pi) * (np.sqrt((x - ext[0]) ** 2 + dy0 + z2)
                           - np.sqrt((x - ext[1]) ** 2 + dy0 + z2))
    dx0 = (x - x0) ** 2
    v = (k_max / np.pi) * (np.sqrt(dx0 + (y - ext[2]) ** 2 + z2)
                           - np.sqrt(dx0 + (y - ext[3]) ** 2 + z2))
    r = _corner_sum(ext, p)
    rad = r * r - _gap(ext)
    if np.any(rad <= _gap(ext) * 1e-12):
        raise OracleDomainError("compressed coordinates undefined")
    n = (k_max / (2.0 * TWO_PI)) * np.sqrt(rad) - (k_min / (2.0 * TWO_PI)) * r
    return np.stack([u, v, n], axis=-1)


# --------------------------------------------------------------------------
# subimage grids (ffbp.py:74-307)
# --------------------------------------------------------------------------

@dataclass
class Grid:
    ext: tuple
    origin: np.ndarray
    step: np.ndarray
    positions: np.ndarray          # [nu, nv, nn, 3]
    valid: np.ndarray              # [nu, nv, nn] bool
    core: tuple
    start: int = 0
    stop: int = 0
    newton_iters: int = 0

    @property
    def dims(self):
        return self.valid.shape

    @property
    def n_valid(self):
        return int(self.valid.sum())

    def core_masked(self):
        sl = tuple(slice(a, b + 1) for a, b in self.core)
        return 1.0 - self.valid[sl].mean()


def _check_core(g: Grid):
    # SubimageGrid.__post_init__ (ffbp.py:119-133)
    masked = g.core_masked()
    if masked >= 0.5:
        raise OracleDomainError(f"{100 * masked:.0f}% of core lattice points have "
                                "no valid inverse position")


@dataclass
class Plan:
    """Lattice metadata of build_subimage_grid before Newton (ffbp.py:237-304)."""
    origin: np.ndarray
    step: np.ndarray
    counts: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    axes: list
    near: list
    core: tuple


def plan_grid(ext, region, k_min, k_max, gamma=1.4, pad=GRID_PAD) -> Plan:
    """The data-independent part of build_subimage_grid: bounds from
    llt_forward on the region's 5^3 boundary lattice (ffbp.py:237-243),
    u/v plane trimming (ffbp.py:248-257), near band (ffbp.py:294-301) and
    core box (ffbp.py:302-304)."""
    b = _bounds(region)
    axes5 = [np.linspace(lo, hi, 5) for lo, hi in b]
    mesh = np.meshgrid(*axes5, indexing="ij")
    uvn = llt_forward(ext, np.stack([m.ravel() for m in mesh], axis=-1), k_min, k_max)
    lo, hi = uvn.min(axis=0), uvn.max(axis=0)
    step = np.full(3, 1.0 / gamma)
    origin = lo - pad * step
    counts = np.ceil((hi - lo) / step).astype(int) + 1 + 2 * pad
    limit = (k_max / np.pi * (ext[1] - ext[0]), k_max / np.pi * (ext[3] - ext[2]))
    for a in (0, 1):  # ffbp.py:248-257 u/v plane trimming
        keep = np.abs(origin[a] + step[a] * np.arange(counts[a])) < limit[a] + 2.0 * step[a]
        if keep.any() and not keep.all():
            first = int(np.argmax(keep))
            last = counts[a] - 1 - int(np.argmax(keep[::-1]))
            origin[a] += first * step[a]
            counts[a] = last - first + 1
    axes = [origin[a] + step[a] * np.arange(counts[a]) for a in range(3)]
    eps = 1e-9 * step
    near = [(axes[a] >= lo[a] - GRID_PAD * step[a] - eps[a])
            & (axes[a] <= hi[a] + GRID_PAD * step[a] + eps[a]) for a in range(3)]
    core = []
    for a in range(3):
        img = (axes[a] >= lo[a] - eps[a]) & (axes[a] <= hi[a] + eps[a])
        core.append((int(np.argmax(img)), int(counts[a] - 1 - np.argmax(img[::-1]))))
    return Plan(origin=origin, step=step, counts=counts, lo=lo, hi=hi, axes=axes, near=near,
                core=tuple(core))


def build_grid(ext, region, k_min, k_max, gamma=1.4, margin=0.25, tol=1e-9,
               max_iter=50, pad=GRID_PAD, start=0, stop=0, prune=False) -> Grid:
    """build_subimage_grid (ffbp.py:179-307) for a lateral extents box.

    ``prune`` skips Newton on (u, v) columns outside the near band, whose
    points end up masked whatever Newton returns; masks and
    valid positions are unchanged, masked positions are left as guesses.
    """
    if not gamma >= 1.0:
        raise OracleConfigError("oversampling factor must be at least 1")
    if region.z_min <= 0.0:
        raise OracleConfigError("region must sit strictly in front of the array")
    b = _bounds(region)
    pl = plan_grid(ext, region, k_min, k_max, gamma, pad)
    origin, step, counts, lo, hi = pl.origin, pl.step, pl.counts, pl.lo, pl.hi
    axes, near, core = pl.axes, pl.near, pl.core
    center = np.array([(b[a, 0] + b[a, 1]) / 2 for a in range(3)])
    extent = b[:, 1] - b[:, 0]
    max_step = 0.5 * float(np.linalg.norm(extent))
    slack = margin * extent + 3.0 * GRID_PAD * step * extent / np.maximum(hi - lo, 1e-12)
    nu, nv, nn = (int(c) for c in counts)

    uu, vv = np.meshgrid(axes[0], axes[1], indexing="ij")
    uu, vv = uu.ravel(), vv.ravel()
    cols = np.arange(nu * nv)
    if prune:
        cols = cols[(near[0][:, None] & near[1][None, :]).ravel()]
    positions = np.broadcast_to(center, (nu * nv, nn, 3)).copy()
    ok_all = np.zeros((nu * nv, nn), dtype=bool)
    guess = np.broadcast_to(center, (cols.size, 3)).copy()
    total_iters = 0
    w_stop = nn if not prune else (int(np.nonzero(near[2])[0].max()) + 1 if near[2].any() else 0)
    for w in range(w_stop):  # ffbp.py:275-282, warm starts along n
        tgt = np.stack([uu[cols], vv[cols], np.full(cols.size, axes[2][w])], axis=-1)
        pos, ok, it = invert_newton(ext, tgt, guess, k_min, k_max, tol, max_iter,
                                    max_step)
        total_iters += int(it.sum())
        positions[cols, w] = pos
        ok_all[cols, w] = ok
        guess = np.where(ok[:, None], pos, center)
    positions = positions.reshape(nu, nv, nn, 3)
    valid = ok_all.reshape(nu, nv, nn).copy()
    for a in range(3):  # inside-slack test, ffbp.py:283-289
        valid &= (positions[..., a] >= b[a, 0] - slack[a]) & (positions[..., a] <= b[a, 1] + slack[a])
    valid &= near[0][:, None, None] & near[1][None, :, None] & near[2][None, None, :]
    g = Grid(ext=tuple(ext), origin=origin, step=step, positions=positions,
             valid=valid, core=tuple(core), start=start, stop=stop,
             newton_iters=total_iters)
    _check_core(g)
    return g


@dataclass
class Sub:
    grid: Grid
    values: np.ndarray              # [nu, nv, nn] complex128, raw (not downconverted)


def level1(prof: Profiles, grid: Grid) -> Sub:
    """level1_reconstruct (ffbp.py:310-340): delay-window mask from the 8
    corners of the leaf's 3-D element bbox, then backproject the leaf."""
    flat = grid.positions.reshape(-1, 3)
    mask = grid.valid.ravel().copy()
    if mask.any():
        els = prof.elements[grid.start:grid.stop]
        lo, hi = els.min(axis=0), els.max(axis=0)
        corners = np.array([np.where(np.array(bits, dtype=bool), hi, lo)
                            for bits in np.ndindex(2, 2, 2)])
        pts = flat[mask]
        dmax = np.sqrt(((pts[:, None, :] - corners[None]) ** 2).sum(-1)).max(axis=1)
        mask[mask] = 2.0 * dmax / C_LIGHT <= prof.window[1]
    if not np.array_equal(mask, grid.valid.ravel()):
        grid = Grid(**{**grid.__dict__, "valid": mask.reshape(grid.dims)})
        _check_core(grid)
    vals = np.zeros(flat.shape[0], dtype=complex)
    if mask.any():
        vals[mask] = backproject(prof, slice(grid.start, grid.stop), flat[mask])
    return Sub(grid=grid, values=vals.reshape(grid.dims))


def merge_onto_points(children, points, k_min, k_max, kernel="linear"):
    """_merge_onto_points (ffbp.py:343-374), N-ary in the children."""
    pts = np.asarray(points, dtype=float)
    total = np.zeros(pts.shape[0], dtype=complex)
    good = np.ones(pts.shape[0], dtype=bool)
    for ch in children:
        g = ch.grid
        coords = (llt_forward(g.ext, pts, k_min, k_max) - g.origin) / g.step
        down = ch.values * np.exp(-1j * sdc_phase(g.ext, g.positions, k_min, k_max))
        val, ok = interpolate(down, coords, kernel)
        total += np.where(ok, val, 0.0) * np.exp(1j * sdc_phase(g.ext, pts, k_min, k_max))
        good &= ok
    total[~good] = 0.0
    return total, int((~good).sum())


def merge_children(children, pgrid: Grid, k_min, k_max, kernel="linear"):
    """merge_pair (ffbp.py:377-412) generalised to N children."""
    for ch in children:
        if not (pgrid.start <= ch.grid.start and ch.grid.stop <= pgrid.stop):
            raise OracleConfigError("children must cover element slices inside "
                                    "the parent subarray")
    flat = pgrid.positions.reshape(-1, 3)
    mask = pgrid.valid.ravel()
    vals = np.zeros(flat.shape[0], dtype=complex)
    flagged = 0
    if mask.any():
        merged, flagged = merge_onto_points(children, flat[mask], k_min, k_max, kernel)
        vals[mask] = merged
    return Sub(grid=pgrid, values=vals.reshape(pgrid.dims)), flagged


def leaf_bounds(n, levels):
    """partition_subarrays split (model.py:377-382)."""
    n_leaves = 2 ** (levels - 1)
    if levels < 1 or n_leaves > n:
        raise OracleConfigError("invalid factorisation depth")
    base, extra = divmod(n, n_leaves)
    sizes = [base + (1 if i < extra else 0) for i in range(n_leaves)]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(int)


def tree_levels(n, levels):
    """List (per level, 1-based level = index + 1) of (start, stop) slices."""
    b = leaf_bounds(n, levels)
    tiers = [list(zip(b[:-1].tolist(), b[1:].tolist()))]
    while len(tiers[-1]) > 1:
        f = tiers[-1]
        tiers.append([(f[2 * i][0], f[2 * i + 1][1]) for i in range(len(f) // 2)])
    return tiers


def grid_levels(levels, merge_factor=2):
    """1-based tree levels that carry subimage grids for a merge factor
    2^s: 1, 1+s, 1+2s, ... below the root (binary: 1..M-1)."""
    s = int(np.log2(merge_factor))
    if 2 ** s != merge_factor or s < 1:
        raise OracleConfigError("merge factor must be a power of two >= 2")
    return list(range(1, levels, s))


def hhffbpa_reconstruct(cube, region, final_dims=None, levels=None, gamma=1.4,
                        kernel="linear", margin=0.25, upsample=8, merge_factor=2,
                        profiles=None, prune=True, keep=None):
    """hhffbpa_reconstruct (ffbp.py:415-513).

    merge_factor=2 is the reference's binary schedule exactly.  merge_factor
    4 (BASELINE configs 0/2/4) is the N-ary harness composed of the same
    primitives: grids only at levels 1, 3, 5, ... and each merge sums four
    children with _merge_onto_points.
    Returns (values, origin, step, provenance); ``keep`` (a dict) receives
    the per-level subimages for inspection.
    """
    _validate(cube, region)
    k_min, k_max = _band(cube.freqs)
    dims = tuple(int(d) for d in (final_dims or default_grid_dims(region, cube.freqs)))
    if levels is None:
        raise OracleConfigError("pass levels explicitly")
    prof = profiles if profiles is not None else range_compress(cube, upsample)
    check_delay_window(prof, region)
    origin, step = region_grid(region, dims)
    cart = _mesh(origin, step, dims)
    n_final = int(np.prod(dims))
    el = prof.elements
    if levels == 1:
        vals = backproject(prof, slice(None), cart)
        level_points, merge_flags, final_flags = [[n_final]], [], 0
    else:
        src_pad = GRID_PAD + (3 if kernel == "cubic" else 2)
        tiers = tree_levels(el.shape[0], levels)
        glev = grid_levels(levels, merge_factor)
        subs = []
        for (a, b) in tiers[0]:
            g = build_grid(extents_of(el, a, b), region, k_min, k_max, gamma, margin,
                           pad=src_pad, start=a, stop=b, prune=prune)
            subs.append(level1(prof, g))
        if keep is not None:
            keep[1] = subs
        level_points = [[s.grid.n_valid for s in subs]]
        merge_flags = []
        for lev in glev[1:]:
            merged, flags = [], 0
            for (a, b) in tiers[lev - 1]:
                kids = [s for s in subs if a <= s.grid.start and s.grid.stop <= b]
                pg = build_grid(extents_of(el, a, b), region, k_min, k_max, gamma,
                                margin, pad=src_pad, start=a, stop=b, prune=prune)
                sub, fl = merge_children(kids, pg, k_min, k_max, kernel)
                merged.append(sub)
                flags += fl
            merge_flags.append(flags)
            level_points.append([s.grid.n_valid for s in merged])
            subs = merged
            if keep is not None:
                keep[lev] = subs
        vals, final_flags = merge_onto_points(subs, cart, k_min, k_max, kernel)
        level_points.append([n_final])
    merged_total = sum(sum(p) for p in level_points[1:])
    flagged_total = sum(merge_flags) + final_flags
    prov = {"algorithm": "hhffbpa", "levels": levels, "gamma": gamma, "kernel": kernel,
            "margin": margin, "upsample": upsample, "dims": list(dims),
            "level_points": [[int(n) for n in p] for p in level_points],
            "merge_flags": [int(f) for f in merge_flags], "final_flags": int(final_flags),
            "flagged_fraction": (flagged_total / merged_total) if merged_total else 0.0}
    if merge_factor != 2:
        prov["merge_factor"] = merge_factor
    return vals.reshape(dims), origin, step, prov
