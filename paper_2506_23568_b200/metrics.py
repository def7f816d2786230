"""Image-quality metrics (reference: metrics.py).

``psnr`` and ``max_intensity_projection`` run on the GPU
(``hhsar_volume_dot`` / ``hhsar_volume_residual`` / ``hhsar_mip``): a 1-2 GB
volume is validated without a host round trip of its samples, and the
``*_device`` forms take device tensors straight from the pipeline
(``DeviceRun.volume``).  ``psf_metrics`` and ``profile_cut`` work on one 1-D
cut (a few hundred samples) on the host, as in the reference.

Same names, arguments, results and exceptions as the reference module
(metrics.py:13-214); volumes are duck-typed (``values``, ``origin``,
``step``, ``same_grid``, ``axis_coords``), so the reference's own
ImageVolume works too.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ConfigError, NumericDomainError

PSNR_SENTINEL_DB = 200.0  # metrics.py:13

_AXIS_NAMES = {"x": 0, "y": 1, "z": 2}


@dataclass(frozen=True)
class PsfReport:
    """Point-spread figures of one 1-D cut (metrics.py:16-43)."""

    mainlobe_width_mm: float
    pslr_db: float
    islr_db: float
    peak_position_m: float

    def to_dict(self) -> dict:
        return {"mainlobe_width_mm": self.mainlobe_width_mm, "pslr_db": self.pslr_db,
                "islr_db": self.islr_db, "peak_position_m": self.peak_position_m}


# ---- GPU volume reductions ------------------------------------------------------

def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.complex64:
        return 0
    if t.dtype == torch.complex128:
        return 1
    raise ConfigError("volume values must be complex64 or complex128")


def _to_device(values, like=None):
    """Host (numpy) or device (torch) complex volume -> contiguous device tensor."""
    import torch
    if isinstance(values, torch.Tensor):
        t = values
        if not t.is_cuda:
            t = t.cuda()
    else:
        a = np.asarray(values)
        if a.dtype not in (np.complex64, np.complex128):
            a = a.astype(np.complex128)
        t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    if like is not None and t.dtype != like.dtype:
        t = t.to(torch.complex128)
    return t.contiguous()


def psnr_device(reference, test) -> float:
    """psnr of two device volumes of equal size (metrics.py:140-150):
    least-squares complex calibration s = vdot(t, r) / vdot(t, t), then
    20 log10(max|r| / rms(s t - r)), clipped at the 200 dB sentinel."""
    import torch
    r, t = reference, test
    if r.dtype != t.dtype:  # compute in the wider type
        r, t = r.to(torch.complex128), t.to(torch.complex128)
    r, t = r.contiguous(), t.contiguous()
    if r.numel() != t.numel():
        raise ConfigError("volumes are on different grids")
    n = r.numel()
    code = _dtype_code(r)
    sums = torch.empty(6, dtype=torch.float64, device=r.device)
    stream = _native.stream_handle()
    _native.call("hhsar_volume_dot", _native.ptr(t), _native.ptr(r), n, code, _native.ptr(sums),
                 stream)
    tt, cr, ci, _, peak = sums[:5].cpu().numpy()
    denom = complex(tt, 0.0)
    scale = complex(cr, ci) / denom if denom != 0 else 0.0
    _native.call("hhsar_volume_residual", _native.ptr(t), _native.ptr(r), n, code,
                 float(scale.real), float(scale.imag), _native.ptr(sums[5:]), stream)
    err2 = float(sums[5].cpu())
    rms = float(np.sqrt(err2 / n)) if n else 0.0
    if rms == 0.0:
        return PSNR_SENTINEL_DB
    return float(min(20.0 * np.log10(float(peak) / rms), PSNR_SENTINEL_DB))


def psnr(reference, test) -> float:
    """Peak signal-to-noise ratio of `test` against `reference` after the
    complex least-squares calibration (metrics.py:126-150)."""
    if not reference.same_grid(test):
        raise ConfigError("volumes are on different grids")
    r = _to_device(reference.values)
    t = _to_device(test.values, like=r)
    if r.dtype != t.dtype:
        r = _to_device(r, like=t)
    return psnr_device(r, t)


def _axis_index(axis) -> int:
    if isinstance(axis, str):
        try:
            return _AXIS_NAMES[axis.lower()]
        except KeyError:
            raise ConfigError(f"axis must be one of x, y, z, got '{axis}'") from None
    idx = int(axis)
    if idx not in (0, 1, 2):
        raise ConfigError(f"axis index must be 0, 1, or 2, got {idx}")
    return idx


def mip_device(values, axis="z", floor_db: float = -40.0):
    """Device [nx, ny, nz] complex tensor -> device float64 projection in
    [0, 1] (metrics.py:170-190)."""
    import torch
    if not floor_db < 0:
        raise ConfigError("floor must be below 0 dB")
    idx = _axis_index(axis)
    v = values.contiguous()
    if v.dim() != 3:
        raise ConfigError("volume values must be a 3-D array")
    dims = np.array(v.shape, dtype=np.int64)
    out_shape = tuple(int(d) for k, d in enumerate(v.shape) if k != idx)
    out = torch.empty(out_shape, dtype=torch.float64, device=v.device)
    _native.call("hhsar_mip", _native.ptr(v), _native.ptr(dims), _dtype_code(v), idx,
                 float(floor_db), _native.ptr(out), _native.stream_handle())
    return out


def max_intensity_projection(volume, axis="z", floor_db: float = -40.0) -> np.ndarray:
    """Per-pixel magnitude maximum along `axis`, dB-scaled to its own peak,
    clipped at `floor_db` and mapped onto [0, 1] (metrics.py:170-190)."""
    if not floor_db < 0:
        raise ConfigError("floor must be below 0 dB")
    _axis_index(axis)
    return mip_device(_to_device(volume.values), axis, floor_db).cpu().numpy()


# ---- 1-D cuts (host, as in the reference) ---------------------------------------

def profile_cut(volume, axis, through) -> tuple[np.ndarray, float]:
    """The 1-D cut along `axis` through the voxel nearest `through`
    (metrics.py:193-214); returns (samples, spacing in metres)."""
    idx = _axis_index(axis)
    through = np.asarray(through, dtype=float).reshape(3)
    sel: list = []
    for a in range(3):
        if a == idx:
            sel.append(slice(None))
        else:
            sel.append(int(np.argmin(np.abs(volume.axis_coords(a) - through[a]))))
    samples = volume.values[tuple(sel)]
    if hasattr(samples, "cpu"):
        samples = samples.cpu().numpy()
    return np.asarray(samples), float(volume.step[idx])


def _null_index(mag: np.ndarray, peak: int, step: int):
    """Index of the first local minimum walking away from the peak: the last
    sample before the magnitude rises again; None if it never rises."""
    run = mag[peak::step] if step > 0 else mag[peak::-1]
    rises = np.flatnonzero(np.diff(run) > 0)
    if rises.size == 0:
        return None
    return peak + step * int(rises[0])


def _half_power_crossing(db: np.ndarray, peak: int, step: int, stop: int) -> float:
    """Fractional index where the profile first reaches -3 dB walking from
    the peak toward `stop`, linear in dB between the straddling samples."""
    idx = np.arange(peak + step, stop + step, step)
    below = np.flatnonzero(db[idx] <= -3.0)
    if below.size == 0:
        raise NumericDomainError("profile never falls 3 dB below its peak inside the mainlobe")
    j = int(idx[below[0]])
    i = j - step
    return i + step * (-3.0 - db[i]) / (db[j] - db[i])


def psf_metrics(profile, spacing: float) -> PsfReport:
    """Mainlobe width (-3 dB), PSLR and ISLR of a 1-D complex profile
    (metrics.py:70-123)."""
    p = np.asarray(profile)
    if p.ndim != 1 or p.size < 5:
        raise ConfigError("profile must be 1-D with at least 5 samples")
    if not spacing > 0:
        raise ConfigError("spacing must be positive")
    mag = np.abs(p).astype(np.float64)
    top = mag.max()
    if top == 0.0:
        raise ConfigError("profile is identically zero")
    at_top = np.flatnonzero(mag == top)
    if at_top.size != 1:
        raise ConfigError("profile peak is not unique")
    peak = int(at_top[0])
    left, right = _null_index(mag, peak, -1), _null_index(mag, peak, +1)
    if left is None or right is None:
        raise NumericDomainError("no null found on at least one side of the peak; the cut is "
                                 "too short to measure")
    with np.errstate(divide="ignore"):
        db = 20.0 * np.log10(mag / top)
    width_m = (_half_power_crossing(db, peak, +1, right)
               - _half_power_crossing(db, peak, -1, left)) * spacing
    main_e = float(np.sum(mag[left:right + 1] ** 2))
    side = np.concatenate([mag[:left], mag[right + 1:]])
    if side.size == 0:
        raise NumericDomainError("no sidelobe region beyond the first nulls")
    side_e = float(np.sum(side ** 2))
    pslr = 20.0 * np.log10(side.max() / top) if side.max() > 0 else -np.inf
    islr = 10.0 * np.log10(side_e / main_e) if side_e > 0 else -np.inf
    return PsfReport(mainlobe_width_mm=width_m * 1e3, pslr_db=float(pslr), islr_db=float(islr),
                     peak_position_m=float(peak * spacing))
