"""TEST INFRASTRUCTURE ONLY -- config-4-scale oracle composed of the
reference's own primitives ("chunked harness").

The reference cannot run BASELINE config 4 as written: its profiles alone
are 137 GB of complex128 (rangecomp.py:91-93).  Three facts of the
reference make a chunked check exact up to summation order:

* range compression is row-independent (rangecomp.py:61-101: one IDFT per
  element row), so each leaf's rows are compressed on their own;
* a subimage grid depends only on its subarray's lateral extents and the
  region (ffbp.py:237-243 bounds from the region's 5^3 boundary lattice,
  Newton per column, ffbp.py:274-282), never on the rest of the aperture;
* _merge_onto_points (ffbp.py:351-374) is pointwise in the evaluation
  points, so a merge or the Cartesian landing can be checked on any subset
  of points given the children's lattices.

``subtree`` rebuilds every leaf and merge of one subtree of the factorised
tree (e.g. one of config 4's eight level-9 subtrees, 1/8 of the aperture)
with oracle.pipeline's restatement of the reference; ``sub_from_lattice``
turns a lattice exported by the device pipeline into the oracle's ``Sub``
so ``merge_onto_points`` can check a merge level or the landing on a point
sample.  Only tests/ and bench.py's parity legs use this module.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .pipeline import (GRID_PAD, Grid, Profiles, Sub, _band, build_grid, extents_of,
                       grid_levels, level1, merge_children, range_compress, sdc_phase,
                       tree_levels)

__all__ = ["SubtreeResult", "subtree", "sub_from_lattice", "raw_values"]


@dataclass
class _Rows:
    """Duck-typed DataCube over a row block (range_compress reads
    .values, .freqs and .aperture.elements)."""
    values: np.ndarray
    freqs: object
    elements: np.ndarray

    @property
    def aperture(self):
        return self


@dataclass
class SubtreeResult:
    levels: dict = field(default_factory=dict)       # grid level -> [Sub] in tree order
    flags: dict = field(default_factory=dict)        # grid level -> [flagged per parent]
    newton_iters: int = 0


def subtree(rows, elements, e0: int, e1: int, freqs, region, levels: int,
            merge_factor: int = 2, upsample: int = 8, gamma: float = 1.4,
            kernel: str = "linear", margin: float = 0.25, row0: int = 0) -> SubtreeResult:
    """Every grid of the factorised tree whose element slice lies inside
    [e0, e1), built and merged as hhffbpa_reconstruct builds them
    (ffbp.py:466-492, the factor-4 schedule per SURVEY Appendix A.3).

    ``rows`` holds cube rows [row0, row0 + len(rows)) (complex64 or 128) and
    must cover [e0, e1); ``elements`` is the FULL aperture (the tree split,
    model.py:352-387, depends on the total element count).  Each leaf's rows
    are range-compressed on their own (rangecomp.py:61-101 is per row), so
    host memory stays at one leaf's complex128 profiles.
    """
    el = np.asarray(elements, dtype=float)
    k_min, k_max = _band(freqs)
    src_pad = GRID_PAD + (3 if kernel == "cubic" else 2)  # ffbp.py:468
    tiers = tree_levels(el.shape[0], levels)
    glev = grid_levels(levels, merge_factor)
    res = SubtreeResult()
    subs = []
    for (a, b) in tiers[0]:
        if not (e0 <= a and b <= e1):
            continue
        prof = range_compress(_Rows(np.asarray(rows[a - row0:b - row0]), freqs, el[a:b]),
                              upsample)
        g = build_grid(extents_of(el, a, b), region, k_min, k_max, gamma, margin,
                       pad=src_pad, start=0, stop=b - a, prune=True)
        res.newton_iters += g.newton_iters
        sub = level1(prof, g)  # leaf-local element indices [0, b - a)
        sub.grid.start, sub.grid.stop = a, b
        subs.append(sub)
    if not subs:
        raise ValueError(f"no leaf lies inside [{e0}, {e1})")
    res.levels[1] = subs
    for lev in glev[1:]:
        parents = [(a, b) for (a, b) in tiers[lev - 1] if e0 <= a and b <= e1]
        if not parents:
            break
        merged, flags = [], []
        for (a, b) in parents:
            kids = [s for s in subs if a <= s.grid.start and s.grid.stop <= b]
            pg = build_grid(extents_of(el, a, b), region, k_min, k_max, gamma, margin,
                            pad=src_pad, start=a, stop=b, prune=True)
            res.newton_iters += pg.newton_iters
            sub, fl = merge_children(kids, pg, k_min, k_max, kernel)
            merged.append(sub)
            flags.append(int(fl))
        res.levels[lev] = merged
        res.flags[lev] = flags
        subs = merged
    return res


def sub_from_lattice(ext, origin, step, dims, core, start, stop, positions, valid,
                     values_down, k_min, k_max, center) -> Sub:
    """Oracle ``Sub`` from a device lattice: positions [P,3] (meaningful at
    valid points), valid [P], values stored DOWNconverted (f' = f
    exp(-j Phi(pos)), ffbp.py:343-348) -> raw values f at valid points, 0
    elsewhere (masked points carry 0, ffbp.py:174-175; their positions are
    set to the region centre, which only enters multiplied by 0)."""
    dims = tuple(int(d) for d in dims)
    valid = np.asarray(valid, dtype=bool).reshape(-1)
    pos = np.where(valid[:, None], np.asarray(positions, dtype=float).reshape(-1, 3),
                   np.asarray(center, dtype=float))
    down = np.asarray(values_down).reshape(-1).astype(np.complex128)
    raw = np.zeros(down.size, dtype=np.complex128)
    raw[valid] = down[valid] * np.exp(1j * sdc_phase(ext, pos[valid], k_min, k_max))
    g = Grid(ext=tuple(float(v) for v in ext), origin=np.asarray(origin, dtype=float).copy(),
             step=np.asarray(step, dtype=float).copy(), positions=pos.reshape(dims + (3,)),
             valid=valid.reshape(dims), core=tuple((int(a), int(b)) for a, b in core),
             start=int(start), stop=int(stop))
    return Sub(grid=g, values=raw.reshape(dims))


def raw_values(ext, positions, values_down, k_min, k_max) -> np.ndarray:
    """Up-converted (raw) values f = f' exp(+j Phi(pos)) of device samples."""
    return np.asarray(values_down).astype(np.complex128) * np.exp(
        1j * sdc_phase(ext, np.asarray(positions, dtype=float), k_min, k_max))
