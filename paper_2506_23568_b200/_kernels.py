"""Operator-level drop-ins for the reference's plugin seam.

The reference selects its three hot loops at import time in
/root/reference/pkg/src/hhsar/_kernels.py (HAVE_NUMBA dispatch, :18-31):
``backproject_gather`` (:98-110), ``lattice_interpolate`` (:354-378) and
``_invert_newton_jit`` (:255-351, called via spectrum.invert_lattice).  This
module offers the same three callables backed by the sm_100a kernels, plus
``install()``, which points an imported ``hhsar`` package at them so the
reference's own pipeline and tests run on the GPU operators.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .bpa import backproject_gather
from .errors import ConfigError

__all__ = ["backproject_gather", "lattice_interpolate", "invert_newton", "install"]


def lattice_interpolate(values, coords, kernel: str = "linear"):
    """(values [nu,nv,nn] complex, coords [n,3]) -> (out complex64 [n], ok bool [n])."""
    import torch
    if kernel not in ("linear", "cubic"):
        raise ConfigError(f"unknown interpolation kernel '{kernel}'")
    _native.library()
    v = np.ascontiguousarray(values, dtype=np.complex64)
    c = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, 3)
    nu, nv, nn = v.shape
    vd = torch.as_tensor(v, device="cuda")
    cd = torch.as_tensor(c, device="cuda")
    out = torch.empty(c.shape[0], dtype=torch.complex64, device="cuda")
    ok = torch.empty(c.shape[0], dtype=torch.uint8, device="cuda")
    _native.call("hhsar_lattice_interp", _native.ptr(vd), nu, nv, nn, _native.ptr(cd),
                 c.shape[0], 0 if kernel == "linear" else 1, _native.ptr(out), _native.ptr(ok),
                 _native.stream_handle())
    return out.cpu().numpy(), ok.cpu().numpy().astype(bool)


def invert_newton(x_min, x_max, y_min, y_max, k_min, k_max, targets, guesses, tol, max_iter,
                  max_step, z_floor):
    """Same signature and results as _invert_newton_jit -> (pos, ok, iters)."""
    import torch
    _native.library()
    t = torch.as_tensor(np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 3),
                        device="cuda")
    g = torch.as_tensor(np.ascontiguousarray(guesses, dtype=np.float64).reshape(-1, 3),
                        device="cuda")
    n = t.shape[0]
    pos = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    ok = torch.empty(n, dtype=torch.uint8, device="cuda")
    it = torch.empty(n, dtype=torch.int64, device="cuda")
    ext = np.array([x_min, x_max, y_min, y_max], dtype=np.float64)
    _native.call("hhsar_invert_newton", _native.ptr(ext), float(k_min), float(k_max),
                 _native.ptr(t), _native.ptr(g), n, float(tol), int(max_iter),
                 float(max_step), float(z_floor), _native.ptr(pos), _native.ptr(ok),
                 _native.ptr(it), _native.stream_handle())
    return pos.cpu().numpy(), ok.cpu().numpy().astype(bool), it.cpu().numpy()


def install(hhsar_module=None):
    """Route an imported reference ``hhsar`` through the GPU operators.

    Patches hhsar._kernels.backproject_gather / lattice_interpolate /
    _invert_newton_jit and the names bpa.py, ffbp.py and spectrum.py bound at
    import time.  Returns a callable that restores the originals.
    """
    import importlib
    h = hhsar_module or importlib.import_module("hhsar")
    k = importlib.import_module(h.__name__ + "._kernels")
    bpa = importlib.import_module(h.__name__ + ".bpa")
    ffbp = importlib.import_module(h.__name__ + ".ffbp")
    spec = importlib.import_module(h.__name__ + ".spectrum")

    def _gather(points, el_pos, envelopes, t0, dt, k_ref):
        v, oow = backproject_gather(points, el_pos, envelopes, t0, dt, k_ref)
        return v.astype(np.complex128), oow

    def _interp(values, coords, kernel="linear"):
        v, ok = lattice_interpolate(values, coords, kernel)
        return v.astype(np.complex128), ok

    saved = [(k, "backproject_gather", k.backproject_gather),
             (k, "lattice_interpolate", k.lattice_interpolate),
             (k, "_invert_newton_jit", k._invert_newton_jit),
             (bpa, "backproject_gather", bpa.backproject_gather),
             (ffbp, "lattice_interpolate", ffbp.lattice_interpolate),
             (spec, "_invert_newton_jit", spec._invert_newton_jit),
             (spec, "HAVE_NUMBA", spec.HAVE_NUMBA)]
    for mod, name in ((k, "backproject_gather"), (bpa, "backproject_gather")):
        setattr(mod, name, _gather)
    for mod, name in ((k, "lattice_interpolate"), (ffbp, "lattice_interpolate")):
        setattr(mod, name, _interp)
    for mod in (k, spec):
        setattr(mod, "_invert_newton_jit", invert_newton)
    spec.HAVE_NUMBA = True  # invert_lattice dispatches on this flag (spectrum.py:365)

    def restore():
        for mod, name, obj in saved:
            setattr(mod, name, obj)
    return restore
