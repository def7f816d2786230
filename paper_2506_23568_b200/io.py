"""Cube / volume files, byte-compatible with the reference formats.

`hhsar-cube-v1` and `hhsar-volume-v1` (/root/reference/pkg/src/hhsar/io.py):
a raw little-endian payload of interleaved float32 real/imaginary pairs plus
a UTF-8 JSON sidecar (same name + ".json").  Cubes are [element][frequency]
with frequency fastest (io.py:85-132); volumes are stored with x fastest
(io.py:135-163).  Reads keep the payload as complex64 (the GPU path's type,
no promotion to complex128) and stage it straight into pinned memory when
CUDA is available, so a reconstruct from file needs one H2D copy.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .errors import ConfigError, IoFormatError
from .model import DataCube, FrequencyGrid, ImagingRegion, SyntheticAperture

CUBE_SCHEMA = "hhsar-cube-v1"
VOLUME_SCHEMA = "hhsar-volume-v1"


def sidecar_path(path) -> Path:
    return Path(str(path) + ".json")


def read_json(path) -> dict:
    """UTF-8 JSON object (io.py:199-211 semantics)."""
    try:
        doc = json.loads(Path(path).read_text(encoding="utf-8"))
    except FileNotFoundError:
        raise
    except OSError as e:
        raise IoFormatError(f"cannot read {path}: {e}") from e
    except json.JSONDecodeError as e:
        raise IoFormatError(f"cannot parse {path}: {e}") from e
    if not isinstance(doc, dict):
        raise IoFormatError(f"{path} must hold a JSON object")
    return doc


def _sidecar(path, schema: str) -> dict:
    side = sidecar_path(path)
    if not side.exists():
        raise IoFormatError(f"missing sidecar {side}")
    try:
        doc = json.loads(side.read_text(encoding="utf-8"))
    except (OSError, json.JSONDecodeError) as e:
        raise IoFormatError(f"cannot parse sidecar {side}: {e}") from e
    if doc.get("schema") != schema:
        raise IoFormatError(f"schema mismatch: expected {schema!r}, found {doc.get('schema')!r}")
    return doc


def _dims(doc: dict, rank: int) -> tuple:
    dims = doc.get("dims")
    if (not isinstance(dims, list) or len(dims) != rank
            or not all(isinstance(d, int) and d > 0 for d in dims)):
        raise IoFormatError(f"dimension mismatch: sidecar dims {dims!r} are not "
                            f"{rank} positive integers")
    return tuple(dims)


def _payload(path, n_values: int) -> np.ndarray:
    """complex64 payload of exactly n_values samples (io.py:52-66 checks)."""
    expected = 8 * n_values
    p = Path(path)
    try:
        size = p.stat().st_size
    except OSError as e:
        raise IoFormatError(f"cannot read payload {path}: {e}") from e
    if size < expected:
        raise IoFormatError(f"truncated payload {path}: expected {expected} bytes, found {size}")
    if size > expected:
        raise IoFormatError(f"dimension mismatch for {path}: sidecar dims imply {expected} "
                            f"bytes, found {size}")
    out = _pinned_empty(n_values)
    with open(p, "rb") as fh:
        fh.readinto(memoryview(out.view(np.uint8)))
    return out


def _pinned_empty(n: int) -> np.ndarray:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.empty(n, dtype=torch.complex64).pin_memory().numpy()
    except Exception:
        pass
    return np.empty(n, dtype=np.complex64)


def region_to_doc(region) -> dict:
    return {"x": [region.x_min, region.x_max], "y": [region.y_min, region.y_max],
            "z": [region.z_min, region.z_max]}


def region_from_doc(doc: dict) -> ImagingRegion:
    try:
        return ImagingRegion(x_min=doc["x"][0], x_max=doc["x"][1], y_min=doc["y"][0],
                             y_max=doc["y"][1], z_min=doc["z"][0], z_max=doc["z"][1])
    except (KeyError, IndexError, TypeError) as e:
        raise IoFormatError(f"malformed region document: {e}") from e


def write_cube(path, cube, region=None, provenance: dict | None = None) -> None:
    """Payload at `path`, sidecar beside it (io.py:85-108)."""
    doc = {"schema": CUBE_SCHEMA,
           "dims": [int(cube.values.shape[0]), int(cube.values.shape[1])],
           "frequencies": {"f_min_hz": cube.freqs.f_min, "f_max_hz": cube.freqs.f_max,
                           "count": cube.freqs.count},
           "aperture": {"nx": cube.aperture.nx, "ny": cube.aperture.ny,
                        "elements": np.asarray(cube.aperture.elements).tolist()}}
    if region is not None:
        doc["region"] = region_to_doc(region)
    if provenance:
        doc["provenance"] = provenance
    Path(path).write_bytes(np.ascontiguousarray(cube.values, dtype="<c8").tobytes())
    sidecar_path(path).write_text(json.dumps(doc, indent=1), encoding="utf-8")


def read_cube(path):
    """(DataCube with complex64 values, region or None) (io.py:111-132)."""
    doc = _sidecar(path, CUBE_SCHEMA)
    n_el, n_f = _dims(doc, 2)
    try:
        f = doc["frequencies"]
        freqs = FrequencyGrid(f_min=float(f["f_min_hz"]), f_max=float(f["f_max_hz"]),
                              count=int(f["count"]))
        a = doc["aperture"]
        aperture = SyntheticAperture(elements=np.asarray(a["elements"], dtype=float),
                                     nx=int(a["nx"]), ny=int(a["ny"]))
    except (KeyError, TypeError, ValueError) as e:
        raise IoFormatError(f"malformed cube sidecar: {e}") from e
    except ConfigError as e:
        raise IoFormatError(f"malformed cube sidecar: {e}") from e
    if freqs.count != n_f or aperture.n_elements != n_el:
        raise IoFormatError(f"dimension mismatch: dims {n_el}x{n_f} disagree with "
                            f"{aperture.n_elements} elements x {freqs.count} frequencies")
    values = _payload(path, n_el * n_f).reshape(n_el, n_f)
    region = region_from_doc(doc["region"]) if "region" in doc else None
    return DataCube(values=values, aperture=aperture, freqs=freqs), region


def write_volume(path, volume) -> None:
    """Payload with x fastest (io.py:135-148)."""
    doc = {"schema": VOLUME_SCHEMA, "dims": [int(d) for d in volume.values.shape],
           "origin": [float(v) for v in volume.origin],
           "step": [float(v) for v in volume.step], "provenance": volume.provenance}
    payload = np.ascontiguousarray(np.asarray(volume.values).transpose(2, 1, 0), dtype="<c8")
    Path(path).write_bytes(payload.tobytes())
    sidecar_path(path).write_text(json.dumps(doc, indent=1), encoding="utf-8")


def read_volume(path):
    """ImageVolume with complex64 values (io.py:151-163)."""
    from .bpa import ImageVolume
    doc = _sidecar(path, VOLUME_SCHEMA)
    dims = _dims(doc, 3)
    try:
        origin = np.asarray(doc["origin"], dtype=float).reshape(3)
        step = np.asarray(doc["step"], dtype=float).reshape(3)
    except (KeyError, TypeError, ValueError) as e:
        raise IoFormatError(f"malformed volume sidecar: {e}") from e
    flat = _payload(path, int(np.prod(dims)))
    values = flat.reshape(dims[2], dims[1], dims[0]).transpose(2, 1, 0)
    return ImageVolume(values=values, origin=origin, step=step,
                       provenance=doc.get("provenance", {}))


# ---- projection images and reports (io.py:166-234 formats) ------------------

_PGM_DEPTHS = {8: (255, ">u1"), 16: (65535, ">u2")}


def export_projection(image, path, depth: int = 8) -> None:
    """A [0, 1] grayscale image (e.g. max_intensity_projection) as a binary
    PGM ("P5"; 16-bit samples big-endian, the format's byte order)."""
    img = np.asarray(image, dtype=np.float64)
    if img.ndim != 2:
        raise ConfigError("projection image must be 2-D")
    if img.size == 0:
        raise ConfigError("projection image is empty")
    if not np.all(np.isfinite(img)) or img.min() < 0.0 or img.max() > 1.0:
        raise ConfigError("projection values must lie in [0, 1]")
    if depth not in _PGM_DEPTHS:
        raise ConfigError("depth must be 8 or 16")
    maxval, dtype = _PGM_DEPTHS[depth]
    pixels = np.floor(img * maxval + 0.5).astype(dtype)
    rows, cols = img.shape
    Path(path).write_bytes(f"P5\n{cols} {rows}\n{maxval}\n".encode("ascii") + pixels.tobytes())


def read_projection(path) -> np.ndarray:
    """A binary PGM back to floats in [0, 1]."""
    raw = Path(path).read_bytes()
    fields = raw.split(b"\n", 3)
    if len(fields) != 4 or fields[0] != b"P5":
        raise IoFormatError(f"{path} is not a binary PGM")
    try:
        cols, rows = (int(v) for v in fields[1].split())
        maxval = int(fields[2])
    except ValueError as e:
        raise IoFormatError(f"malformed PGM header in {path}: {e}") from e
    wide = maxval >= 256
    n = cols * rows * (2 if wide else 1)
    if len(fields[3]) < n:
        raise IoFormatError(f"truncated PGM payload in {path}")
    pixels = np.frombuffer(fields[3][:n], dtype=">u2" if wide else ">u1")
    return pixels.reshape(rows, cols).astype(np.float64) / maxval


def write_report(path, report: dict) -> None:
    """A key-value report as indented, key-sorted JSON (UTF-8)."""
    Path(path).write_text(json.dumps(report, indent=1, sort_keys=True), encoding="utf-8")
