"""BASELINE INFRASTRUCTURE ONLY -- the reference's own CPU path timed on a
bounded, extrapolated sample of BASELINE config 4, and whole at config 3.

Config 4 cannot run through the reference as written (its complex128
profiles alone are 137 GB), so the reference arm times the
unmodified reference functions (``oracle.reference.load()``: the staged
``hhsar`` package, Numba kernels) on pieces of the config-4 tree and
scales each piece by how often it occurs in one volume:

* a level-5 subtree (1/128 of the aperture: 16 leaves of 1,024 elements):
  ``range_compress`` of its 16,384 rows (rangecomp.py:61-101),
  ``build_subimage_grid`` + ``level1_reconstruct`` per leaf
  (ffbp.py:179-340), and the 4 + 1 factor-4 merges through
  ``_merge_onto_points`` (ffbp.py:351-374) onto freshly built parent grids
  -- x 128 subtrees;
* the merges above it (levels 7, 9, 11): one parent per level, its grid and
  its four children's grids built with ``build_subimage_grid`` (build time
  x grids at that level) and the merge through ``_merge_onto_points``
  (x parents at that level);
* the Cartesian landing (ffbp.py:493-495) on one z-slice of the
  1024 x 1024 x 256 grid from the two level-11 subimages -- x 256 slices.

Everything measured is reference code on config-4 geometry; only the
extrapolation is ours.  The leaf/merge cost is data-independent (SURVEY
Appendix C), so sample rows may be a seeded random cube.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

LEAF = 1024            # elements per leaf (2,097,152 / 2,048)
SUBTREE = 16 * LEAF    # a level-5 subtree
GRID_LEVELS = (1, 3, 5, 7, 9, 11)


def _to_ref(hh, w):
    """The workload's geometry as the reference's own types."""
    freqs = hh.FrequencyGrid(float(w.freqs.f_min), float(w.freqs.f_max), int(w.freqs.count))
    r = w.region
    region = hh.ImagingRegion(float(r.x_min), float(r.x_max), float(r.y_min), float(r.y_max),
                              float(r.z_min), float(r.z_max))
    return freqs, region


def _subaperture(hh, elements, a, b, nx=32):
    el = np.ascontiguousarray(np.asarray(elements)[a:b], dtype=float)
    return hh.SyntheticAperture(elements=el, nx=nx, ny=el.shape[0] // nx)


@dataclass
class Config4Sample:
    """Per-piece reference timings (seconds) and the extrapolated volume time."""
    subtree_s: list = field(default_factory=list)       # rc + 16 leaves + 4 + 1 merges
    rc_s: list = field(default_factory=list)            # part of subtree_s
    landing_slice_s: list = field(default_factory=list)
    merge_s: dict = field(default_factory=dict)         # level -> [s]
    build_s: dict = field(default_factory=dict)         # level -> [s per grid build]
    warmup_s: float = 0.0

    def volume_seconds(self) -> float:
        counts = {7: 32, 9: 8, 11: 2}
        t = 128 * float(np.mean(self.subtree_s)) + 256 * float(np.mean(self.landing_slice_s))
        for lev, n in counts.items():
            t += n * (float(np.mean(self.build_s[lev])) + float(np.mean(self.merge_s[lev])))
        return t

    def summary(self) -> dict:
        return {
            "subtree_s": round(float(np.mean(self.subtree_s)), 3),
            "range_compression_16384_rows_s": round(float(np.mean(self.rc_s)), 3),
            "landing_slice_s": round(float(np.mean(self.landing_slice_s)), 3),
            "grid_build_s": {k: round(float(np.mean(v)), 3) for k, v in self.build_s.items()},
            "merge_s": {k: round(float(np.mean(v)), 3) for k, v in self.merge_s.items()},
            "extrapolated_volume_s": round(self.volume_seconds(), 2),
            "formula": "128 x subtree + 32/8/2 x (grid build + merge) at levels 7/9/11 "
                       "+ 256 x landing z-slice",
        }


class Config4Reference:
    """Reference-code sampler for config 4 (merge factor 4, M = 12)."""

    def __init__(self, hh, w, rows_fn):
        """``rows_fn(a, b)`` -> complex cube rows [a, b) of the config."""
        self.hh, self.w, self.rows_fn = hh, w, rows_fn
        self.freqs, self.region = _to_ref(hh, w)
        self.el = np.asarray(w.aperture.elements, dtype=float)
        self.sample = Config4Sample()
        self.upper = {}
        self.tops = None
        self._step = 0

    # -- pieces ------------------------------------------------------------
    def _grid(self, a, b, ap=None, off=0):
        hh = self.hh
        ap = ap if ap is not None else self._full
        return hh.build_subimage_grid(ap, hh.Subarray(a - off, b - off), self.region, self.freqs,
                                      gamma=1.4, margin=0.25, pad=4)

    def _random_sub(self, grid, rng):
        hh = self.hh
        v = (rng.standard_normal(grid.dims) + 1j * rng.standard_normal(grid.dims))
        return hh.ffbp.Subimage(grid=grid, values=np.where(grid.valid, v, 0.0),
                                downconverted=False)

    def _merge(self, kids, pg):
        hh = self.hh
        flat = pg.positions.reshape(-1, 3)
        mask = pg.valid.ravel()
        vals = np.zeros(flat.shape[0], dtype=complex)
        if mask.any():
            vals[mask], _ = hh.ffbp._merge_onto_points(tuple(kids), flat[mask], self.freqs,
                                                       "linear")
        return hh.ffbp.Subimage(grid=pg, values=vals.reshape(pg.dims), downconverted=False)

    def subtree(self, index: int) -> None:
        """Level-5 subtree ``index`` (0..127) through the reference."""
        hh = self.hh
        a = index * SUBTREE
        rows = self.rows_fn(a, a + SUBTREE)  # input fetch: not reference work
        t0 = time.perf_counter()
        ap = _subaperture(hh, self.el, a, a + SUBTREE)
        cube = hh.DataCube(values=rows, aperture=ap, freqs=self.freqs)
        prof = hh.range_compress(cube, upsample=self.w.upsample)
        t1 = time.perf_counter()
        subs = []
        for k in range(16):
            leaf = hh.Subarray(k * LEAF, (k + 1) * LEAF)
            g = hh.build_subimage_grid(ap, leaf, self.region, self.freqs, gamma=1.4, margin=0.25,
                                       pad=4)
            subs.append(hh.level1_reconstruct(prof, leaf, g))
        for span in (4 * LEAF, 16 * LEAF):
            parents = []
            for p in range(SUBTREE // span):
                pg = hh.build_subimage_grid(ap, hh.Subarray(p * span, (p + 1) * span),
                                            self.region, self.freqs, gamma=1.4, margin=0.25,
                                            pad=4)
                parents.append(self._merge(subs[4 * p:4 * p + 4], pg))
            subs = parents
        t2 = time.perf_counter()
        self.sample.rc_s.append(t1 - t0)
        self.sample.subtree_s.append(t2 - t0)

    def prepare_upper(self, seed: int = 4) -> None:
        """Grids of one parent per level 7 / 9 / 11 and of its four children
        (timed per build), plus the second level-11 grid for the landing."""
        hh = self.hh
        rng = np.random.default_rng(seed)
        self._full = hh.SyntheticAperture(elements=self.el, nx=32, ny=self.el.shape[0] // 32)
        t_all = time.perf_counter()
        builds = {5: [], 7: [], 9: [], 11: []}
        for lev in (7, 9, 11):
            span = LEAF << (lev - 1)
            cspan = span // 4
            kids = []
            for c in range(4):
                t = time.perf_counter()
                g = self._grid(c * cspan, (c + 1) * cspan)
                builds[lev - 2].append(time.perf_counter() - t)
                kids.append(self._random_sub(g, rng))
            t = time.perf_counter()
            pg = self._grid(0, span)
            builds[lev].append(time.perf_counter() - t)
            self.upper[lev] = (kids, pg)
        span = LEAF << 10
        t = time.perf_counter()
        g2 = self._grid(span, 2 * span)
        builds[11].append(time.perf_counter() - t)
        pg11 = self.upper[11][1]
        self.tops = (self._random_sub(pg11, rng), self._random_sub(g2, rng))
        self.sample.build_s = {lev: builds[lev] for lev in (7, 9, 11)}
        self.sample.warmup_s = time.perf_counter() - t_all

    def upper_merge(self, lev: int) -> None:
        kids, pg = self.upper[lev]
        t = time.perf_counter()
        self._merge(kids, pg)
        self.sample.merge_s.setdefault(lev, []).append(time.perf_counter() - t)

    def landing_slice(self, iz: int) -> None:
        hh = self.hh
        nx, ny, nz = self.w.dims
        origin, step = hh.bpa.region_grid(self.region, self.w.dims)
        ix, iy = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
        pts = np.stack([origin[0] + step[0] * ix.ravel(), origin[1] + step[1] * iy.ravel(),
                        np.full(ix.size, origin[2] + step[2] * iz)], axis=-1)
        t = time.perf_counter()
        hh.ffbp._merge_onto_points(self.tops, pts, self.freqs, "linear")
        self.sample.landing_slice_s.append(time.perf_counter() - t)

    # -- one bounded step ----------------------------------------------------
    def step(self) -> float:
        """One sample: a subtree, one upper merge, one landing slice; returns
        its wall time."""
        j = self._step
        self._step += 1
        t = time.perf_counter()
        self.subtree((j * 37) % 128)
        self.upper_merge((7, 9, 11)[j % 3])
        self.landing_slice((j * 53) % self.w.dims[2])
        return time.perf_counter() - t

    def complete(self) -> bool:
        return all(lev in self.sample.merge_s for lev in (7, 9, 11))

    def fill(self) -> None:
        """Merges of the levels no step has sampled yet (untimed steps)."""
        for lev in (7, 9, 11):
            if lev not in self.sample.merge_s:
                self.upper_merge(lev)


def warm_jit(hh) -> None:
    """The reference's own JIT warm-up (cli.py:357-362): one tiny
    reconstruction compiles every Numba kernel before anything is timed
    (nothing to compile for the oracle port)."""
    if getattr(hh, "PORT", False):
        return
    ap = hh.SyntheticAperture(elements=np.column_stack([
        np.repeat(np.linspace(-0.01, 0.01, 4), 4), np.tile(np.linspace(-0.01, 0.01, 4), 4),
        np.zeros(16)]), nx=4, ny=4)
    freqs = hh.FrequencyGrid(77e9, 81e9, 8)
    rng = np.random.default_rng(0)
    cube = hh.DataCube(values=rng.standard_normal((16, 8)) + 0j, aperture=ap, freqs=freqs)
    region = hh.ImagingRegion.from_center((0.0, 0.0, 0.2), (0.02, 0.02, 0.02))
    hh.bpa_reconstruct(cube, region, dims=(5, 5, 5), upsample=2)
    hh.hhffbpa_reconstruct(cube, region, (5, 5, 5), hh.FfbpParams(levels=2), upsample=2)
    for kern in ("linear", "cubic"):
        hh.hhffbpa_reconstruct(cube, region, (5, 5, 5), hh.FfbpParams(levels=2, kernel=kern),
                               upsample=2)
