"""TEST / BASELINE INFRASTRUCTURE ONLY -- the oracle port behind the subset
of the reference package's API that oracle/refarm.py drives.

bench.py times the reference's own CPU path (the unmodified ``hhsar``
staged in oracle/_ref) whenever it is present; where it is not (a box that
received the repo without the staged copy), the reference arm and the CPU
baseline fall back to this restatement (``kind: "port"``): the same
sampler, the same pieces, computed by oracle/pipeline.py (numpy + the OpenMP
C loops), each function citing the reference code it restates there.
"""

from __future__ import annotations

from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np

from . import pipeline as op

PORT = True  # marks this module as the fallback (not the reference package)


@dataclass(frozen=True)
class FrequencyGrid:
    f_min: float
    f_max: float
    count: int


@dataclass(frozen=True)
class ImagingRegion:
    x_min: float
    x_max: float
    y_min: float
    y_max: float
    z_min: float
    z_max: float


@dataclass(frozen=True)
class SyntheticAperture:
    elements: np.ndarray
    nx: int
    ny: int

    @property
    def n_elements(self) -> int:
        return int(np.asarray(self.elements).shape[0])


@dataclass(frozen=True)
class Subarray:
    start: int
    stop: int


@dataclass(frozen=True)
class DataCube:
    values: np.ndarray
    aperture: SyntheticAperture
    freqs: FrequencyGrid


@dataclass(frozen=True)
class FfbpParams:
    levels: int | None = None
    gamma: float = 1.4
    kernel: str = "linear"
    margin: float = 0.25


def range_compress(cube, upsample=8):
    """rangecomp.py:61-101 (oracle.pipeline.range_compress)."""
    return op.range_compress(cube, upsample)


def build_subimage_grid(aperture, subarray, region, freqs, gamma=1.4, margin=0.25, pad=2):
    """ffbp.py:179-307 (oracle.pipeline.build_grid; pruned Newton, exact masks)."""
    k_min, k_max = op._band(freqs)
    ext = op.extents_of(aperture.elements, subarray.start, subarray.stop)
    return op.build_grid(ext, region, k_min, k_max, gamma, margin, pad=pad,
                         start=subarray.start, stop=subarray.stop, prune=True)


def level1_reconstruct(profiles, subarray, grid):
    """ffbp.py:310-340 (oracle.pipeline.level1)."""
    return op.level1(profiles, grid)


def _merge_onto_points(children, points, freqs, kernel):
    """ffbp.py:351-374 (oracle.pipeline.merge_onto_points)."""
    k_min, k_max = op._band(freqs)
    return op.merge_onto_points(children, points, k_min, k_max, kernel)


def _subimage(grid, values, downconverted=False):
    return op.Sub(grid=grid, values=np.asarray(values))


ffbp = SimpleNamespace(_merge_onto_points=_merge_onto_points, Subimage=_subimage)
bpa = SimpleNamespace(region_grid=op.region_grid)


def hhffbpa_reconstruct(cube, region, dims, params, upsample=8):
    """ffbp.py:415-513 (oracle.pipeline.hhffbpa_reconstruct)."""
    vals, _, _, prov = op.hhffbpa_reconstruct(cube, region, dims, levels=params.levels,
                                              gamma=params.gamma, kernel=params.kernel,
                                              margin=params.margin, upsample=upsample)
    return SimpleNamespace(values=vals, provenance=prov)


def bpa_reconstruct(cube, region, dims=None, upsample=8):
    vals, _, _, prov = op.bpa_reconstruct(cube, region, dims, upsample)
    return SimpleNamespace(values=vals, provenance=prov)
