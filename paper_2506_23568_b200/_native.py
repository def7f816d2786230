"""ctypes binding of libhhsar_b200.so (the C ABI in include/hhsar_b200.h).

PyTorch supplies device memory and the CUDA stream; every call passes raw
device pointers (``tensor.data_ptr()``) plus the current stream handle.  There
is no CPU fallback: if the library or a CUDA device is missing, the first call
raises NativeUnavailableError.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import NativeUnavailableError

LIB_NAME = "libhhsar_b200.so"
# HHSAR_LIB overrides the in-tree library (A/B builds in tools/, never set
# by the tests or the bench)
LIB_PATH = Path(os.environ.get("HHSAR_LIB") or Path(__file__).resolve().parent / LIB_NAME)

# numpy mirrors of the C structs (align=True follows the C layout rules;
# checked against hhsar_abi_layout() at load time)
GEOM_DTYPE = np.dtype([
    ("region", "<f8", 6), ("center", "<f8", 3), ("k_min", "<f8"), ("k_max", "<f8"),
    ("c_uv", "<f8"), ("c_nhi", "<f8"), ("c_nlo", "<f8"), ("step", "<f8"),
    ("margin", "<f8"), ("max_step", "<f8"), ("tol", "<f8"), ("z_floor", "<f8"),
    ("window_hi", "<f8"), ("pad", "<i4"), ("max_iter", "<i4")], align=True)

GRID_DTYPE = np.dtype([
    ("ext", "<f8", 4), ("box", "<f8", 6), ("lo", "<f8", 3), ("hi", "<f8", 3),
    ("origin", "<f8", 3), ("slack_lo", "<f8", 3), ("slack_hi", "<f8", 3),
    ("dims", "<i4", 3), ("near_lo", "<i4", 3), ("near_hi", "<i4", 3),
    ("core_lo", "<i4", 3), ("core_hi", "<i4", 3), ("is_leaf", "<i4"),
    ("act_lo", "<i4", 2), ("act_hi", "<i4", 2), ("start", "<i8"), ("stop", "<i8"), ("leaf_lo", "<i8"), ("leaf_hi", "<i8"),
    ("offset", "<i8"), ("col_offset", "<i8")], align=True)

GRID_STATS = 6

_P, _I64, _I32, _D, _F = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                          ctypes.c_double, ctypes.c_float)

# name -> argtypes (restype int status unless noted)
SIGNATURES = {
    "hhsar_last_error": ([], ctypes.c_char_p),
    "hhsar_version": ([], ctypes.c_int),
    "hhsar_device_sm_count": ([], ctypes.c_int),
    "hhsar_abi_layout": ([_P, _I32], ctypes.c_int),
    "hhsar_bp_gather": ([_P, _I64, _P, _I64, _P, _I64, _D, _D, _D, _P, _P, _P], ctypes.c_int),
    "hhsar_lattice_interp": ([_P, _I64, _I64, _I64, _P, _I64, _I32, _P, _P, _P], ctypes.c_int),
    "hhsar_invert_newton": ([_P, _D, _D, _P, _P, _I64, _D, _I32, _D, _D, _P, _P, _P, _P],
                            ctypes.c_int),
    "hhsar_bpa_cartesian": ([_P, _P, _P, _I64, _I64, _P, _I64, _P, _I64, _D, _D, _D, _P, _P, _P],
                            ctypes.c_int),
    "hhsar_range_pad": ([_P, _I64, _I64, _I64, _P, _P], ctypes.c_int),
    "hhsar_range_demod": ([_P, _I64, _I64, _D, _D, _F, _P], ctypes.c_int),
    "hhsar_range_compress": ([_P, _I64, _I64, _I64, _D, _D, _P, _P], ctypes.c_int),
    "hhsar_range_compress_window": ([_P, _I64, _I64, _I64, _D, _D, _I64, _I64, _P, _P],
                                    ctypes.c_int),
    "hhsar_leaf_boxes": ([_P, _P, _I64, _P, _P], ctypes.c_int),
    "hhsar_grid_plan": ([_P, _I64, _P, _P, _I64, _P, _P, _P, _P], ctypes.c_int),
    "hhsar_leaf_range_gate": ([_P, _I64, _P, _D, _I64, _P, _P], ctypes.c_int),
    "hhsar_grid_newton": ([_P, _I64, _I64, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "hhsar_volume_dot": ([_P, _P, _I64, _I32, _P, _P], ctypes.c_int),
    "hhsar_volume_residual": ([_P, _P, _I64, _I32, _D, _D, _P, _P], ctypes.c_int),
    "hhsar_mip": ([_P, _P, _I32, _I32, _D, _P, _P], ctypes.c_int),
    "hhsar_leaf_bp": ([_P, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _D, _D, _D, _P, _I32,
                       _P, _P, _P], ctypes.c_int),
    "hhsar_merge_level": ([_P, _I64, _I64, _P, _P, _P, _I64, _I32, _P, _P, _I32, _I32, _P, _P,
                           _P], ctypes.c_int),
    "hhsar_downconvert": ([_P, _I64, _I64, _P, _P, _P, _P, _P], ctypes.c_int),
    "hhsar_merge_cartesian": ([_P, _P, _P, _I64, _I64, _P, _I64, _P, _I64, _I64, _P, _I32, _P,
                               _P, _P],
                              ctypes.c_int),
    "hhsar_simulate": ([_P, _I64, _P, _P, _I64, _P, _I64, _P, _P], ctypes.c_int),
    "hhsar_simulate_uniform": ([_P, _I64, _P, _P, _I64, _D, _D, _I64, _P, _P], ctypes.c_int),
}

_lib = None


def library(require_gpu: bool = True):
    """Load (once) and return the ctypes handle; fail loudly if unusable."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeUnavailableError(
                f"{LIB_PATH} is missing; build it with __graft_entry__.build() "
                "(make -C paper_2506_23568_b200/csrc)")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is None and os.environ.get("HHSAR_LIB"):
                continue  # an older A/B build
            if fn is None:
                raise NativeUnavailableError(f"{LIB_PATH} does not export {name}")
            fn.argtypes = args
            fn.restype = res
        _check_layout(lib)
        _lib = lib
    if require_gpu:
        import torch
        if not torch.cuda.is_available():
            raise NativeUnavailableError("no CUDA device visible: the hot path has no CPU "
                                         "fallback")
    return _lib


def _check_layout(lib) -> None:
    out = np.zeros(16, dtype=np.int64)
    n = lib.hhsar_abi_layout(out.ctypes.data, 16)
    want = [GEOM_DTYPE.itemsize, GRID_DTYPE.itemsize, GEOM_DTYPE.fields["window_hi"][1],
            GEOM_DTYPE.fields["pad"][1], GRID_DTYPE.fields["dims"][1],
            GRID_DTYPE.fields["is_leaf"][1], GRID_DTYPE.fields["start"][1],
            GRID_DTYPE.fields["offset"][1], GRID_DTYPE.fields["col_offset"][1]]
    if n != len(want) or list(out[:n]) != want:
        raise NativeUnavailableError(f"ABI layout mismatch: library {list(out[:n])} vs "
                                     f"binding {want}")


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


_fns = {}


def call(name: str, *args) -> None:
    """Invoke an entry point; raise RuntimeError with the library's message
    on a non-zero status (argument errors are pre-validated by callers)."""
    fn = _fns.get(name)
    if fn is None:
        fn = _fns[name] = getattr(library(), name)
    status = fn(*args)
    if status != 0:
        msg = library().hhsar_last_error().decode(errors="replace")
        raise RuntimeError(f"{name} failed (status {status}): {msg}")


def stream_handle(stream=None):
    """cudaStream_t of `stream` (default: torch's current stream on the
    current device, read without constructing a Stream object)."""
    if stream is not None:
        return ctypes.c_void_p(stream.cuda_stream)
    import torch
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))


def ptr(t) -> ctypes.c_void_p:
    """Device (or host numpy) pointer of a contiguous tensor/array."""
    if isinstance(t, np.ndarray):
        return ctypes.c_void_p(t.ctypes.data)
    if t is None:
        return ctypes.c_void_p(0)
    if not t.is_contiguous():
        raise ValueError("kernel arguments must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def host_struct(dtype, values: dict) -> np.ndarray:
    a = np.zeros(1, dtype=dtype)
    for k, v in values.items():
        a[k] = v
    return a


def device_struct(arr: np.ndarray, device="cuda"):
    """Copy a structured numpy array to the device as raw bytes."""
    import torch
    raw = torch.from_numpy(np.ascontiguousarray(arr).view(np.uint8).reshape(-1))
    return raw.to(device, non_blocking=False)


def simulate(elements, positions, refl, k_samples, device="cuda"):
    """Born cube on the device (hhsar_simulate); returns a complex64 tensor."""
    import torch
    library()
    el = torch.tensor(np.asarray(elements, dtype=np.float64), device=device)
    pos = torch.tensor(np.asarray(positions, dtype=np.float64).reshape(-1, 3), device=device)
    r = np.ascontiguousarray(np.asarray(refl, dtype=np.complex128))
    rr = torch.as_tensor(r.view(np.float64), device=device)
    k = torch.as_tensor(np.ascontiguousarray(k_samples, dtype=np.float64), device=device)
    out = torch.empty((el.shape[0], k.shape[0]), dtype=torch.complex64, device=device)
    call("hhsar_simulate", ptr(el), el.shape[0], ptr(pos), ptr(rr), pos.shape[0],
         ptr(k), k.shape[0], ptr(out), stream_handle())
    return out


def simulate_uniform(elements, positions, refl, freqs, device="cuda", out=None):
    """Born cube on the device for a uniform FrequencyGrid
    (hhsar_simulate_uniform: fp32 phasor recurrence, float64 seeds) --
    the generator for the large configs; complex64 tensor [N_el, n_f]
    (written into ``out`` when given, e.g. a row slice of a bigger cube)."""
    import torch
    library()
    if isinstance(elements, torch.Tensor):
        el = elements.to(device=device, dtype=torch.float64).contiguous()
    else:
        el = torch.as_tensor(np.ascontiguousarray(elements, dtype=np.float64), device=device)
    pos = torch.tensor(np.asarray(positions, dtype=np.float64).reshape(-1, 3), device=device)
    r = np.ascontiguousarray(np.asarray(refl, dtype=np.complex128))
    rr = torch.as_tensor(r.view(np.float64), device=device)
    n_f = int(freqs.count)
    k0 = float(freqs.k_min)
    dk = (float(freqs.k_max) - k0) / (n_f - 1) if n_f > 1 else 0.0
    if out is None:
        out = torch.empty((el.shape[0], n_f), dtype=torch.complex64, device=device)
    call("hhsar_simulate_uniform", ptr(el), el.shape[0], ptr(pos), ptr(rr), pos.shape[0], k0,
         dk, n_f, ptr(out), stream_handle())
    return out


def visible() -> bool:
    """True when the library loads and a CUDA device is present."""
    try:
        library()
        return True
    except Exception:
        return False


os.environ.setdefault("CUDA_MODULE_LOADING", "LAZY")


def c_void_p_offset(t, k: int) -> ctypes.c_void_p:
    """Pointer to element k of a contiguous device tensor."""
    return ctypes.c_void_p(t.data_ptr() + int(k) * t.element_size())
