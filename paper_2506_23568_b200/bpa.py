"""Direct backprojection (BPA) on the GPU: the drop-in for hhsar.bpa.

Entry points keep the reference signatures (/root/reference/pkg/src/hhsar/
bpa.py): ``bpa_reconstruct(cube, region, dims=None, upsample=8)``,
``backproject(profiles, elements, points)``, ``region_grid``,
``check_delay_window`` and the ``ImageVolume`` result type, with the same
exceptions and messages.  The voxel x element sum runs in
hhsar_bpa_cartesian (csrc/bp.cu) over device-resident complex64 envelopes.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ConfigError, NumericDomainError
from .model import C_LIGHT, Subarray, validate_geometry
from .rangecomp import RangeProfileSet, range_compress


@dataclass(frozen=True)
class ImageVolume:
    """Complex samples on a uniform Cartesian grid (bpa.py:22-70).

    ``values`` is [nx, ny, nz] (z fastest).  The GPU path returns complex64
    (the arithmetic type of the kernels and of the volume file format);
    complex128 input is kept as is.
    """

    values: np.ndarray
    origin: np.ndarray
    step: np.ndarray
    provenance: dict = field(default_factory=dict)

    def __post_init__(self):
        v = np.asarray(self.values)
        if not (np.iscomplexobj(v) and v.dtype in (np.complex64, np.complex128)):
            v = v.astype(np.complex128)
        if v.ndim != 3:
            raise ConfigError("volume values must be a 3-D array")
        if not getattr(self, "_finite_checked", False) and not np.all(np.isfinite(v)):
            raise ConfigError("volume values must be finite")
        object.__setattr__(self, "values", v)
        object.__setattr__(self, "origin", np.asarray(self.origin, dtype=float))
        object.__setattr__(self, "step", np.asarray(self.step, dtype=float))

    @classmethod
    def _trusted(cls, values, origin, step, provenance):
        """Build from values already checked finite on the device."""
        obj = cls.__new__(cls)
        object.__setattr__(obj, "_finite_checked", True)
        cls.__init__(obj, values, origin, step, provenance)
        return obj

    @property
    def dims(self):
        return self.values.shape

    def axis_coords(self, axis: int) -> np.ndarray:
        return self.origin[axis] + self.step[axis] * np.arange(self.dims[axis])

    def grid_points(self) -> np.ndarray:
        g = np.meshgrid(*(self.axis_coords(a) for a in range(3)), indexing="ij")
        return np.stack([a.ravel() for a in g], axis=-1)

    def same_grid(self, other) -> bool:
        return (tuple(self.dims) == tuple(other.dims)
                and np.allclose(self.origin, other.origin, atol=1e-12)
                and np.allclose(self.step, other.step, atol=1e-12))


def region_grid(region, dims):
    """Edge-to-edge uniform grid (bpa.py:73-83), bit-identical float64."""
    dims = tuple(int(d) for d in dims)
    if len(dims) != 3 or any(d < 1 for d in dims):
        raise ConfigError("grid dims must be three integers >= 1")
    los = np.array([region.x_min, region.y_min, region.z_min])
    his = np.array([region.x_max, region.y_max, region.z_max])
    d = np.array(dims)
    origin = np.where(d > 1, los, (los + his) / 2)
    step = np.where(d > 1, (his - los) / np.maximum(d - 1, 1), his - los)
    return origin, step


def default_grid_dims(region, freqs):
    """Resolution-limit grid (spectrum.py:534-545)."""
    rates = (np.pi / (2.0 * freqs.k_max), np.pi / (2.0 * freqs.k_max), np.pi / freqs.k_max)
    ext = (region.x_max - region.x_min, region.y_max - region.y_min, region.z_max - region.z_min)
    return tuple(int(round(e / r)) + 1 for e, r in zip(ext, rates))


def _corners(region) -> np.ndarray:
    return np.array([(x, y, z) for x in (region.x_min, region.x_max)
                     for y in (region.y_min, region.y_max)
                     for z in (region.z_min, region.z_max)])


def check_delay_window(profiles, region) -> None:
    """Farthest element-to-region-corner delay vs the profile window
    (bpa.py:130-141).  Evaluated on the device when positions live there."""
    el_dev = getattr(profiles, "elements_dev", None)
    if el_dev is not None:
        import torch
        c = torch.as_tensor(_corners(region), device=el_dev.device)
        d2 = ((el_dev[:, None, :] - c[None]) ** 2).sum(-1).max()
        d_max = float(np.sqrt(float(d2)))
    else:
        el = np.asarray(profiles.aperture.elements)
        d_max = float(np.linalg.norm(_corners(region)[None] - el[:, None], axis=2).max())
    tau_max = 2.0 * d_max / C_LIGHT
    lo, hi = profiles.window
    if tau_max > hi or 0.0 < lo:
        raise NumericDomainError(
            f"max round-trip delay {tau_max:.3e} s exceeds the alias-free "
            f"profile window [{lo:.3e}, {hi:.3e}]; the frequency step is too "
            "coarse for this geometry")


def _selection(profiles, elements):
    """Resolve a Subarray / slice / index array (bpa.py:86-94) to a device
    index range or index tensor."""
    n = profiles.envelopes.shape[0]
    if isinstance(elements, Subarray) or (hasattr(elements, "start") and hasattr(elements, "stop")
                                          and not isinstance(elements, slice)):
        return slice(int(elements.start), int(elements.stop))
    if isinstance(elements, slice):
        return slice(*elements.indices(n)[:2]) if elements.step in (None, 1) else elements
    return np.asarray(elements, dtype=np.int64)


def el_f32x4(el_dev):
    """float64 [N,3] device positions -> float32 [N,4] (x, y, z, 0)."""
    import torch
    out = torch.zeros((el_dev.shape[0], 4), dtype=torch.float32, device=el_dev.device)
    out[:, :3] = el_dev
    return out


def backproject(profiles: RangeProfileSet, elements, points) -> np.ndarray:
    """Backproject a subset of elements onto arbitrary points (bpa.py:97-127).

    Returns a host complex64 array; raises NumericDomainError when any
    point-element delay falls outside the profile window.
    """
    import torch
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    sel = _selection(profiles, elements)
    if isinstance(sel, slice):
        el = profiles.elements_dev[sel]
        env = profiles.envelopes[sel]
    else:
        idx = torch.as_tensor(sel, device=profiles.envelopes.device)
        el = profiles.elements_dev[idx]
        env = profiles.envelopes[idx]
    if el.shape[0] == 0:
        return np.zeros(pts.shape[0], dtype=np.complex64)
    values, oow = backproject_gather(pts, el, env, profiles.t0, profiles.dt, profiles.k_ref)
    bad = int(oow.sum())
    if bad:
        raise NumericDomainError(
            f"{bad} point-element delays fell outside the profile window; "
            "enlarge the upsampled profile or shrink the geometry")
    return values


def backproject_gather(points, el_pos, envelopes, t0, dt, k_ref):
    """Operator-level drop-in for _kernels.backproject_gather
    (_kernels.py:98-110): returns (values complex64 [n], oow int64 [n])."""
    import torch
    _native.library()
    dev = envelopes.device if isinstance(envelopes, torch.Tensor) else torch.device("cuda")
    pts = torch.as_tensor(np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
                          if not isinstance(points, torch.Tensor) else points, device=dev,
                          dtype=torch.float64).contiguous()
    el = torch.as_tensor(el_pos if isinstance(el_pos, torch.Tensor)
                         else np.ascontiguousarray(el_pos, dtype=np.float64),
                         device=dev, dtype=torch.float64).reshape(-1, 3).contiguous()
    env = torch.as_tensor(envelopes if isinstance(envelopes, torch.Tensor)
                          else np.ascontiguousarray(envelopes), device=dev).to(torch.complex64)
    env = env.contiguous()
    n = pts.shape[0]
    out = torch.empty(n, dtype=torch.complex64, device=dev)
    oow = torch.empty(n, dtype=torch.int64, device=dev)
    _native.call("hhsar_bp_gather", _native.ptr(pts), n, _native.ptr(el), el.shape[0],
                 _native.ptr(env), env.shape[1], float(t0), float(dt), float(k_ref),
                 _native.ptr(out), _native.ptr(oow), _native.stream_handle())
    return out.cpu().numpy(), oow.cpu().numpy()


def bpa_volume_device(env, el4, region, dims, t0, dt, k_ref, vox_range=None, out=None,
                      oow=None):
    """Device-resident direct BPA over region_grid voxels [vb, ve) -> complex64
    tensor (flat).  ``oow`` (int64[1] device) accumulates out-of-window hits."""
    import torch
    origin, step = region_grid(region, dims)
    total = int(np.prod(dims))
    vb, ve = vox_range if vox_range is not None else (0, total)
    if out is None:
        out = torch.empty(ve - vb, dtype=torch.complex64, device=env.device)
    if oow is None:
        oow = torch.zeros(1, dtype=torch.int64, device=env.device)
    d = np.asarray(dims, dtype=np.int64)
    _native.call("hhsar_bpa_cartesian", _native.ptr(np.ascontiguousarray(origin)),
                 _native.ptr(np.ascontiguousarray(step)), _native.ptr(d), vb, ve,
                 _native.ptr(el4), el4.shape[0], _native.ptr(env), env.shape[1], float(t0),
                 float(dt), float(k_ref), _native.ptr(out), _native.ptr(oow),
                 _native.stream_handle())
    return out, oow


def bpa_reconstruct(cube, region, dims=None, upsample: int = 8) -> ImageVolume:
    """Full-aperture BPA onto a uniform Cartesian grid (bpa.py:144-176)."""
    validate_geometry(cube.aperture, region)
    if dims is None:
        dims = default_grid_dims(region, cube.freqs)
    dims = tuple(int(d) for d in dims)
    origin, step = region_grid(region, dims)
    profiles = range_compress(cube, upsample)
    check_delay_window(profiles, region)
    vol, oow = bpa_volume_device(profiles.envelopes, el_f32x4(profiles.elements_dev), region,
                                 dims, profiles.t0, profiles.dt, profiles.k_ref)
    return _finish(vol, oow, dims, origin, step,
                   {"algorithm": "bpa", "upsample": upsample, "dims": list(dims)})[0]


def _finish(vol, oow, dims, origin, step, provenance, extra_flags=None):
    """One device->host round trip for the volume, the finiteness flag and
    the out-of-window count, then the reference's error semantics."""
    import torch
    finite = torch.isfinite(torch.view_as_real(vol)).all().reshape(1).to(torch.int64)
    scalars = torch.cat([oow.reshape(-1)[:1], finite] +
                        ([extra_flags.reshape(-1)] if extra_flags is not None else []))
    # pinned destinations (the caching host allocator reuses them across
    # calls) so both copies are DMA transfers queued behind the kernels; one
    # stream synchronisation for everything
    host_t = torch.empty(vol.shape, dtype=vol.dtype, pin_memory=True)
    sc_t = torch.empty(scalars.shape, dtype=scalars.dtype, pin_memory=True)
    host_t.copy_(vol, non_blocking=True)
    sc_t.copy_(scalars, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    host = host_t.numpy().reshape(dims)
    sc = sc_t.numpy()
    if int(sc[0]):
        raise NumericDomainError(
            f"{int(sc[0])} point-element delays fell outside the profile window; "
            "enlarge the upsampled profile or shrink the geometry")
    if not int(sc[1]):
        raise ConfigError("volume values must be finite")
    return ImageVolume._trusted(host, origin, step, provenance), sc[2:]
