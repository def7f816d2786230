"""Geometry and configuration types consumed by the reconstruct entry points.

Host-side mirror of the reference types the hot path reads
(/root/reference/pkg/src/hhsar/model.py, simulator.py:20-38).  Every entry
point in this package duck-types its arguments, so the reference's own
objects (``hhsar.DataCube``, ``hhsar.ImagingRegion`` ...) are accepted
unchanged; these classes exist so the package also runs where the reference
is not installed (the GPU box).

Only geometry metadata lives here; echo data goes straight to HBM.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError

C_LIGHT = 299792458.0  # model.py:20


def _frozen(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    a.setflags(write=False)
    return a


@dataclass(frozen=True)
class FrequencyGrid:
    """Equidistant stepped-frequency band (model.py:30-70)."""

    f_min: float
    f_max: float
    count: int

    def __post_init__(self):
        if not (self.f_min > 0 and np.isfinite(self.f_min)
                and np.isfinite(self.f_max)):
            raise ConfigError("frequency band edges must be positive and finite")
        if self.f_min >= self.f_max:
            raise ConfigError("f_min must be strictly below f_max")
        if int(self.count) != self.count or self.count < 2:
            raise ConfigError("frequency count must be an integer >= 2")

    @property
    def frequencies(self) -> np.ndarray:
        return np.linspace(self.f_min, self.f_max, self.count)

    @property
    def k_samples(self) -> np.ndarray:
        return 2.0 * np.pi * self.frequencies / C_LIGHT

    @property
    def k_min(self) -> float:
        return 2.0 * np.pi * self.f_min / C_LIGHT

    @property
    def k_max(self) -> float:
        return 2.0 * np.pi * self.f_max / C_LIGHT


@dataclass(frozen=True)
class SyntheticAperture:
    """Ordered phase-centre positions (model.py:91-145); nx*ny == n."""

    elements: np.ndarray
    nx: int
    ny: int

    def __post_init__(self):
        e = np.asarray(self.elements, dtype=float)
        if e.ndim != 2 or e.shape[1] != 3 or e.shape[0] == 0:
            raise ConfigError("aperture needs a non-empty (n, 3) element array")
        if not np.all(np.isfinite(e)):
            raise ConfigError("aperture element coordinates must be finite")
        if self.nx * self.ny != e.shape[0]:
            raise ConfigError("scan lattice shape does not match element count")
        object.__setattr__(self, "elements", _frozen(e))

    @property
    def n_elements(self) -> int:
        return self.elements.shape[0]

    @property
    def x_min(self) -> float:
        return float(self.elements[:, 0].min())

    @property
    def x_max(self) -> float:
        return float(self.elements[:, 0].max())

    @property
    def y_min(self) -> float:
        return float(self.elements[:, 1].min())

    @property
    def y_max(self) -> float:
        return float(self.elements[:, 1].max())

    @property
    def z_max(self) -> float:
        return float(self.elements[:, 2].max())


@dataclass(frozen=True)
class ImagingRegion:
    """Axis-aligned box in front of the aperture (model.py:148-219)."""

    x_min: float
    x_max: float
    y_min: float
    y_max: float
    z_min: float
    z_max: float

    def __post_init__(self):
        for lo, hi, ax in ((self.x_min, self.x_max, "x"),
                           (self.y_min, self.y_max, "y"),
                           (self.z_min, self.z_max, "z")):
            if not (np.isfinite(lo) and np.isfinite(hi) and lo < hi):
                raise ConfigError(f"region {ax} extent must be positive and finite")

    @classmethod
    def from_center(cls, center, extents) -> "ImagingRegion":
        (cx, cy, cz), (ex, ey, ez) = center, extents
        return cls(cx - ex / 2, cx + ex / 2, cy - ey / 2, cy + ey / 2,
                   cz - ez / 2, cz + ez / 2)

    @property
    def extents(self):
        return (self.x_max - self.x_min, self.y_max - self.y_min,
                self.z_max - self.z_min)

    @property
    def center(self):
        return ((self.x_min + self.x_max) / 2, (self.y_min + self.y_max) / 2,
                (self.z_min + self.z_max) / 2)

    @property
    def volume(self) -> float:
        ex, ey, ez = self.extents
        return ex * ey * ez

    @property
    def diagonal(self) -> float:
        return float(np.linalg.norm(self.extents))

    def corners(self) -> np.ndarray:
        return np.array([(x, y, z) for x in (self.x_min, self.x_max)
                         for y in (self.y_min, self.y_max)
                         for z in (self.z_min, self.z_max)])

    def boundary_lattice(self, per_axis: int = 5) -> np.ndarray:
        return boundary_lattice(self, per_axis)

    def contains(self, points, margin: float = 0.0) -> np.ndarray:
        p = np.asarray(points, dtype=float)
        ok = np.ones(p.shape[:-1], dtype=bool)
        for a, (lo, hi) in enumerate(region_bounds(self)):
            m = margin * (hi - lo)
            ok &= (p[..., a] >= lo - m) & (p[..., a] <= hi + m)
        return ok


def region_bounds(region) -> tuple:
    """((x_min, x_max), (y_min, y_max), (z_min, z_max)) of any region-like."""
    return ((region.x_min, region.x_max), (region.y_min, region.y_max),
            (region.z_min, region.z_max))


def boundary_lattice(region, per_axis: int = 5) -> np.ndarray:
    """per_axis^3 ij-ordered lattice over the box (model.py:199-209).

    Built with np.linspace exactly like the reference so the lattice bounds
    derived from it (ffbp.py:237-240) are bit-identical.
    """
    axes = [np.linspace(lo, hi, per_axis) for lo, hi in region_bounds(region)]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=-1)


@dataclass(frozen=True)
class DataCube:
    """Measured s(p', k) indexed [element, frequency] (simulator.py:20-38).

    Unlike the reference (which promotes to complex128), complex64 payloads
    are kept as complex64: the GPU path computes in complex64 and the cube
    file format is complex64 on disk (io.py:85-108).
    """

    values: np.ndarray
    aperture: SyntheticAperture
    freqs: FrequencyGrid

    def __post_init__(self):
        v = np.asarray(self.values)
        if not np.iscomplexobj(v) or v.dtype not in (np.complex64, np.complex128):
            v = v.astype(np.complex128)
        expected = (self.aperture.n_elements, self.freqs.count)
        if v.shape != expected:
            raise ConfigError(f"cube shape {v.shape} does not match "
                              f"aperture x frequency shape {expected}")
        object.__setattr__(self, "values", _frozen(v))


@dataclass(frozen=True)
class Subarray:
    """Contiguous element slice [start, stop) (model.py:311-324)."""

    start: int
    stop: int

    @property
    def size(self) -> int:
        return self.stop - self.start

    @property
    def indices(self) -> np.ndarray:
        return np.arange(self.start, self.stop)


@dataclass(frozen=True)
class SubarrayTree:
    """Binary merge hierarchy; levels[0] holds the 2^(M-1) leaves."""

    aperture: SyntheticAperture
    levels: tuple = field(default_factory=tuple)

    @property
    def depth(self) -> int:
        return len(self.levels)

    def children(self, level: int, index: int):
        if level < 2:
            raise ConfigError("level-1 subarrays have no children")
        finer = self.levels[level - 2]
        return finer[2 * index], finer[2 * index + 1]


def leaf_bounds(n_elements: int, levels: int) -> np.ndarray:
    """Start offsets (length 2^(M-1)+1) of the balanced contiguous leaves.

    Same split as model.py:377-382: the first n mod L leaves get one extra
    element.
    """
    if levels < 1:
        raise ConfigError("levels must be at least 1")
    n_leaves = 1 << (levels - 1)
    if n_leaves > n_elements:
        raise ConfigError(f"{levels} levels need at least {n_leaves} elements, "
                          f"aperture has {n_elements}")
    base, extra = divmod(n_elements, n_leaves)
    sizes = np.full(n_leaves, base, dtype=np.int64)
    sizes[:extra] += 1
    return np.concatenate([[0], np.cumsum(sizes)])


def partition_subarrays(aperture, levels: int) -> SubarrayTree:
    """Binary subarray hierarchy (model.py:352-387)."""
    bounds = leaf_bounds(aperture.n_elements, levels)
    tiers = [tuple(Subarray(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:]))]
    while len(tiers[-1]) > 1:
        f = tiers[-1]
        tiers.append(tuple(Subarray(f[2 * i].start, f[2 * i + 1].stop)
                           for i in range(len(f) // 2)))
    return SubarrayTree(aperture=aperture, levels=tuple(tiers))


@dataclass(frozen=True)
class JitterSpec:
    """Handheld trajectory uncertainty (model.py:73-88)."""

    depth_amplitude: float = 0.0
    lateral_sigma: float = 0.0

    def __post_init__(self):
        if self.depth_amplitude < 0 or self.lateral_sigma < 0:
            raise ConfigError("jitter amplitudes must be non-negative")


def generate_handheld_aperture(nx: int, ny: int, extent: float, jitter=None,
                               seed: int = 0) -> SyntheticAperture:
    """Jittered raster scan (model.py:256-308), same seeded draws: lateral
    Gaussian noise, then a box-smoothed random walk in z' scaled to the
    depth bound."""
    if nx < 1 or ny < 1:
        raise ConfigError("aperture lattice shape must be at least 1x1")
    if not (extent > 0 and np.isfinite(extent)):
        raise ConfigError("aperture extent must be positive")
    jitter = jitter or JitterSpec()
    xs = np.linspace(-extent / 2, extent / 2, nx) if nx > 1 else np.zeros(1)
    ys = np.linspace(-extent / 2, extent / 2, ny) if ny > 1 else np.zeros(1)
    gx, gy = np.meshgrid(xs, ys)
    n = nx * ny
    el = np.zeros((n, 3))
    el[:, 0], el[:, 1] = gx.ravel(), gy.ravel()
    rng = np.random.default_rng(seed)
    if jitter.lateral_sigma > 0:
        el[:, :2] += rng.normal(0.0, jitter.lateral_sigma, (n, 2))
    if jitter.depth_amplitude > 0:
        walk = np.cumsum(rng.standard_normal(n))
        w = max(3, nx)
        walk = np.convolve(np.pad(walk, w, mode="edge"), np.ones(w) / w, "same")[w:-w]
        walk -= walk.mean()
        peak = np.abs(walk).max()
        if peak > 0:
            el[:, 2] = walk * (jitter.depth_amplitude / peak)
    return SyntheticAperture(elements=el, nx=nx, ny=ny)


@dataclass(frozen=True)
class Scene:
    """Point scatterers (model.py:222-245)."""

    positions: np.ndarray
    reflectivity: np.ndarray

    def __post_init__(self):
        p = np.atleast_2d(np.asarray(self.positions, dtype=float))
        if p.size == 0:
            p = p.reshape(0, 3)
        r = np.atleast_1d(np.asarray(self.reflectivity, dtype=complex))
        if p.ndim != 2 or p.shape[1] != 3:
            raise ConfigError("scene positions must have shape (n, 3)")
        if r.shape != (p.shape[0],):
            raise ConfigError("one reflectivity per scatterer required")
        if p.size and not np.all(np.isfinite(p)):
            raise ConfigError("scatterer positions must be finite")
        object.__setattr__(self, "positions", _frozen(p))
        object.__setattr__(self, "reflectivity", _frozen(r))

    @property
    def n_scatterers(self) -> int:
        return self.positions.shape[0]


def scene_grid(shape, spacing: float, center, reflectivity: complex = 1.0) -> Scene:
    """Regular scatterer lattice (simulator.py:72-94)."""
    shape = tuple(int(s) for s in shape)
    if any(s < 1 for s in shape):
        raise ConfigError("grid shape entries must be at least 1")
    if spacing < 0:
        raise ConfigError("grid spacing must be non-negative")
    axes = [(np.arange(s) - (s - 1) / 2) * spacing + c for s, c in zip(shape, center)]
    g = np.meshgrid(*axes, indexing="ij")
    pos = np.stack([a.ravel() for a in g], axis=-1)
    return Scene(pos, np.full(pos.shape[0], reflectivity, dtype=complex))


def scene_star(diameter: float, spokes: int, points_per_spoke: int, center,
               reflectivity: complex = 1.0) -> Scene:
    """Radial-spoke target (simulator.py:97-113)."""
    if diameter <= 0 or spokes < 1 or points_per_spoke < 1:
        raise ConfigError("star needs positive diameter, spokes, and density")
    radii = np.linspace(diameter / (2 * (points_per_spoke + 1)), diameter / 2,
                        points_per_spoke)
    ang = np.arange(spokes) * (2 * np.pi / spokes)
    cx, cy, cz = center
    pos = np.array([(cx + r * np.cos(a), cy + r * np.sin(a), cz) for a in ang for r in radii])
    return Scene(pos, np.full(pos.shape[0], reflectivity, dtype=complex))


def scene_from_spec(spec: dict, region=None) -> Scene:
    """Scene from a config mapping (simulator.py:116-161): kinds grid, star,
    points; every scatterer must lie inside ``region`` when given."""
    if not isinstance(spec, dict) or "kind" not in spec:
        raise ConfigError("scene spec must be a mapping with a 'kind' entry")
    kind = spec["kind"]
    known = {"grid": {"kind", "shape", "spacing", "center", "reflectivity"},
             "star": {"kind", "diameter", "spokes", "points_per_spoke", "center",
                      "reflectivity"},
             "points": {"kind", "positions", "reflectivity"}}
    if kind not in known:
        raise ConfigError(f"unknown scene kind '{kind}'")
    unknown = set(spec) - known[kind]
    if unknown:
        raise ConfigError(f"unknown scene fields: {sorted(unknown)}")
    try:
        if kind == "grid":
            scene = scene_grid(spec["shape"], spec["spacing"], spec["center"],
                               complex(spec.get("reflectivity", 1.0)))
        elif kind == "star":
            scene = scene_star(spec["diameter"], spec["spokes"], spec["points_per_spoke"],
                               spec["center"], complex(spec.get("reflectivity", 1.0)))
        else:
            pos = np.asarray(spec["positions"], dtype=float)
            refl = spec.get("reflectivity", [1.0] * len(pos))
            if np.isscalar(refl):
                refl = [refl] * len(pos)
            scene = Scene(pos, np.asarray(refl, dtype=complex))
    except KeyError as exc:
        raise ConfigError(f"scene spec missing field {exc}") from exc
    if region is not None and scene.n_scatterers:
        inside = region.contains(scene.positions)
        if not np.all(inside):
            bad = scene.positions[~inside][0]
            raise ConfigError(f"scatterer at {tuple(bad)} lies outside the imaging region")
    return scene


def validate_geometry(aperture, region) -> None:
    """Region must sit strictly in front of every element (model.py:248-253)."""
    z_max = float(np.asarray(aperture.elements)[:, 2].max())
    if region.z_min <= z_max:
        raise ConfigError(f"region z_min {region.z_min:g} must exceed the deepest "
                          f"aperture element z' {z_max:g}")
