"""Host-side pieces of the analytic spectrum geometry (spectrum.py in the
reference).  The per-point maps -- llt_forward (Eq. 37), sdc_phase (Eq. 30)
and the Newton inversion -- run inside the CUDA kernels (csrc/common.cuh,
csrc/grid.cu); this module keeps the small value types the API exposes."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

TWO_PI = 2.0 * np.pi


@dataclass(frozen=True)
class SubarrayExtents:
    """Lateral bbox of a subarray's elements, z' ignored (spectrum.py:33-69)."""

    x_min: float
    x_max: float
    y_min: float
    y_max: float

    def __post_init__(self):
        if self.x_min > self.x_max or self.y_min > self.y_max:
            raise ConfigError("subarray extents need min <= max per axis")

    @classmethod
    def from_aperture(cls, aperture, subarray=None) -> "SubarrayExtents":
        e = np.asarray(aperture.elements)
        if subarray is not None:
            e = e[subarray.start:subarray.stop]
        return cls(float(e[:, 0].min()), float(e[:, 0].max()),
                   float(e[:, 1].min()), float(e[:, 1].max()))

    @property
    def dx(self) -> float:
        return self.x_max - self.x_min

    @property
    def dy(self) -> float:
        return self.y_max - self.y_min

    def as_tuple(self):
        return (self.x_min, self.x_max, self.y_min, self.y_max)


def default_grid_dims(region, kgrid) -> tuple:
    """Reconstruction grid at the band's resolution limits (spectrum.py:534-545)."""
    rates = (np.pi / (2.0 * kgrid.k_max), np.pi / (2.0 * kgrid.k_max), np.pi / kgrid.k_max)
    ext = (region.x_max - region.x_min, region.y_max - region.y_min, region.z_max - region.z_min)
    return tuple(int(round(e / r)) + 1 for e, r in zip(ext, rates))
