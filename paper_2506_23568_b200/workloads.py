"""Seeded synthetic workloads for the five BASELINE.json configurations.

BASELINE.json's configs use features the reference does not model (MIMO
arrays, freehand trajectories, noise, merge factor 4); SURVEY.md Appendix A
maps each onto the reference's monostatic, contiguous-leaf semantics and this
module implements that mapping:

* MIMO "a Tx x b Rx" -> a*b monostatic phase centres at 2 mm pitch
  (simulator.py:64-68 is monostatic);
* freehand trajectory -> per axis a sum of 3 sinusoids normalised to the
  stated amplitude plus 0.5 mm Gaussian jitter; elements frame-major;
* config 0 raster -> 32x32 jittered raster in Morton 4x4-block order so the
  16-element leaves are the 4x4 blocks;
* noise -> complex AWGN at the stated SNR, added before complex64
  quantisation.

The draw order from ``np.random.default_rng(seed)`` is fixed: trajectory,
jitter, scene positions, reflectivities, noise.  Geometry is host numpy; the
echo cube of the large configs is produced by the CUDA Born simulator
(``simulate_cube``), small ones may use the numpy path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .model import (C_LIGHT, DataCube, FrequencyGrid, ImagingRegion,
                    SyntheticAperture)


@dataclass
class Workload:
    name: str
    aperture: SyntheticAperture
    freqs: FrequencyGrid
    region: ImagingRegion
    dims: tuple
    upsample: int
    scene_pos: np.ndarray
    scene_refl: np.ndarray
    snr_db: float | None
    seed: int
    levels: int | None = None
    merge_factor: int = 2
    algorithm: str = "bpa"
    notes: dict = field(default_factory=dict)

    @property
    def n_elements(self) -> int:
        return self.aperture.n_elements

    @property
    def n_voxels(self) -> int:
        return int(np.prod(self.dims))

    @property
    def bpa_units(self) -> float:
        """voxel x aperture-element backprojections of one direct BPA."""
        return float(self.n_voxels) * float(self.n_elements)


def _morton4(bx: np.ndarray, by: np.ndarray) -> np.ndarray:
    code = np.zeros_like(bx)
    for bit in range(8):
        code |= ((bx >> bit) & 1) << (2 * bit)
        code |= ((by >> bit) & 1) << (2 * bit + 1)
    return code


def raster_morton(n_side: int, extent: float, jitter: float, rng, block: int = 4):
    """Jittered n x n raster (x fast, y slow: model.py:288-294) reordered
    block-major so each contiguous run of block^2 elements is one block, blocks
    in Morton order (binary siblings are spatial neighbours)."""
    xs = np.linspace(-extent / 2, extent / 2, n_side)
    gx, gy = np.meshgrid(xs, xs)
    el = np.zeros((n_side * n_side, 3))
    el[:, 0], el[:, 1] = gx.ravel(), gy.ravel()
    el[:, :2] += rng.uniform(-jitter, jitter, (el.shape[0], 2))
    iy, ix = np.divmod(np.arange(el.shape[0]), n_side)
    bx, by = ix // block, iy // block
    inner = (iy % block) * block + (ix % block)
    order = np.lexsort((inner, _morton4(bx, by)))
    return el[order]


def freehand(n_frames: int, amplitudes, rng, jitter: float = 0.5e-3):
    """Smooth freehand path: per axis a weighted sum of 3 sinusoids over
    t in [0, 1] (U(0.3, 2.0) cycles, U(0, 2pi) phases, U(0.5, 1) weights)
    normalised so its peak equals the axis amplitude, plus Gaussian jitter."""
    t = np.linspace(0.0, 1.0, n_frames)
    path = np.zeros((n_frames, 3))
    for a, amp in enumerate(amplitudes):
        f = rng.uniform(0.3, 2.0, 3)
        ph = rng.uniform(0.0, 2 * np.pi, 3)
        w = rng.uniform(0.5, 1.0, 3)
        s = (w[None] * np.sin(2 * np.pi * f[None] * t[:, None] + ph[None])).sum(1)
        path[:, a] = s * (amp / np.abs(s).max())
    path += rng.normal(0.0, jitter, path.shape)
    return path


def virtual_array(nx: int, ny: int, pitch: float = 2e-3) -> np.ndarray:
    """nx x ny phase-centre offsets (x fast), centred on the frame origin."""
    ox = (np.arange(nx) - (nx - 1) / 2) * pitch
    oy = (np.arange(ny) - (ny - 1) / 2) * pitch
    gx, gy = np.meshgrid(ox, oy)
    return np.stack([gx.ravel(), gy.ravel(), np.zeros(nx * ny)], axis=-1)


def frames_to_elements(path: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """Frame-major element list: element f*n_v + k = path[f] + offsets[k]."""
    return (path[:, None, :] + offsets[None, :, :]).reshape(-1, 3)


def config(index: int, *, frames: int | None = None) -> Workload:
    """The BASELINE.json configuration ``index`` (0-4), seeded 1000+index.

    ``frames`` shrinks the trajectory for tests (same generator, fewer frames).
    """
    seed = 1000 + index
    rng = np.random.default_rng(seed)
    if index == 0:
        el = raster_morton(32, 0.1, 1e-3, rng)
        ap = SyntheticAperture(elements=el, nx=32, ny=32)
        freqs = FrequencyGrid(77e9, 81e9, 64)
        g = (np.arange(3) - 1) * 0.02
        gx, gy = np.meshgrid(g, g, indexing="ij")
        pos = np.stack([gx.ravel(), gy.ravel(), np.full(9, 0.25)], axis=-1)
        refl = np.ones(9, dtype=complex)
        region = ImagingRegion.from_center((0.0, 0.0, 0.25),
                                           (63 * 1.5e-3, 63 * 1.5e-3, 31 * 3e-3))
        return Workload("config0", ap, freqs, region, (64, 64, 32), 8, pos, refl, 30.0,
                        seed, levels=7, merge_factor=4, algorithm="hhffbpa")
    if index in (1, 2):
        nf = frames or 4000
        path = freehand(nf, (0.05, 0.04, 0.005), rng)
        el = frames_to_elements(path, virtual_array(1, 8))
        ap = SyntheticAperture(elements=el, nx=8, ny=nf)
        freqs = FrequencyGrid(77e9, 81e9, 256)
        pos = np.column_stack([rng.uniform(-0.075, 0.075, 200), rng.uniform(-0.075, 0.075, 200),
                               rng.uniform(0.275, 0.325, 200)])
        refl = rng.rayleigh(1.0, 200).astype(complex)
        region = ImagingRegion.from_center((0.0, 0.0, 0.3), (0.199, 0.199, 0.126))
        w = Workload(f"config{index}", ap, freqs, region, (200, 200, 64), 4, pos, refl, None,
                     seed, algorithm="bpa" if index == 1 else "hhffbpa")
        if index == 2:
            w.levels = 9
        return w
    if index == 3:
        nf = frames or 16384
        path = freehand(nf, (0.12, 0.10, 0.01), rng)
        el = frames_to_elements(path, virtual_array(1, 8))
        ap = SyntheticAperture(elements=el, nx=8, ny=nf)
        freqs = FrequencyGrid(77e9, 81e9, 512)
        x = rng.uniform(-0.15, 0.15, 5000)
        y = rng.uniform(-0.15, 0.15, 5000)
        pos = np.column_stack([x, y, 0.3 + 0.02 * np.sin(20 * x) * np.cos(15 * y)])
        refl = (rng.normal(size=5000) + 1j * rng.normal(size=5000)) / np.sqrt(2)
        region = ImagingRegion.from_center((0.0, 0.0, 0.3), (0.3066, 0.3066, 0.1905))
        return Workload("config3", ap, freqs, region, (512, 512, 128), 4, pos, refl, None,
                        seed, levels=11, algorithm="hhffbpa")
    if index == 4:
        nf = frames or 65536
        path = freehand(nf, (0.2, 0.2, 0.01), rng)
        el = frames_to_elements(path, virtual_array(4, 8))
        ap = SyntheticAperture(elements=el, nx=32, ny=nf)
        freqs = FrequencyGrid(75e9, 85e9, 1024)
        layers = []
        for z0 in (0.32, 0.35, 0.38):
            x = rng.uniform(-0.14, 0.14, 20000 // 3 + 1)
            y = rng.uniform(-0.14, 0.14, x.size)
            layers.append(np.column_stack([x, y, z0 + 0.01 * np.sin(15 * x) * np.cos(12 * y)]))
        pos = np.concatenate(layers)[:20000]
        refl = (rng.normal(size=20000) + 1j * rng.normal(size=20000)) / np.sqrt(2)
        region = ImagingRegion.from_center((0.0, 0.0, 0.35), (0.3, 0.3, 0.1))
        return Workload("config4", ap, freqs, region, (1024, 1024, 256), 4, pos, refl, None,
                        seed, levels=12, merge_factor=4, algorithm="hhffbpa")
    raise ValueError(f"no config {index}")


def simulate_numpy(w: Workload, rng=None) -> DataCube:
    """First-order Born cube (simulator.py:41-69) in float64 numpy, plus the
    workload's noise, quantised to complex64.  For small workloads."""
    el = np.asarray(w.aperture.elements)
    k = w.freqs.k_samples
    vals = np.zeros((el.shape[0], k.size), dtype=complex)
    for p, s in zip(w.scene_pos, w.scene_refl):
        d = np.linalg.norm(el - p, axis=1)
        vals += s * np.exp(-2j * np.outer(d, k))
    return DataCube(values=add_noise(vals, w, rng), aperture=w.aperture, freqs=w.freqs)


def add_noise(vals: np.ndarray, w: Workload, rng=None) -> np.ndarray:
    """Complex AWGN at w.snr_db (per-sample mean power), then complex64."""
    if w.snr_db is not None:
        rng = rng or np.random.default_rng(w.seed + 7)
        sigma = np.sqrt(np.mean(np.abs(vals) ** 2) / 10 ** (w.snr_db / 10) / 2)
        vals = vals + sigma * (rng.normal(size=vals.shape) + 1j * rng.normal(size=vals.shape))
    return np.ascontiguousarray(vals, dtype=np.complex64)


def simulate_cube(w: Workload, device="cuda") -> DataCube:
    """Born cube on the GPU (CUDA kernel hhsar_simulate, float64 phases) with
    the workload's noise; returns a host complex64 DataCube."""
    import torch
    from . import _native
    vals = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                            w.freqs.k_samples, device=device)
    host = vals.cpu().numpy()
    return DataCube(values=add_noise(host, w), aperture=w.aperture, freqs=w.freqs)


def delay_bin_size(w: Workload) -> float:
    """Range-bin pitch in metres of one-way distance, c*dt/2."""
    k_min, k_max = w.freqs.k_min, w.freqs.k_max
    n_t = w.upsample * w.freqs.count
    dt = 2.0 * np.pi / (n_t * ((k_max - k_min) / (w.freqs.count - 1)) * C_LIGHT)
    return C_LIGHT * dt / 2
