"""Load the reference-generated golden cases (tests/golden/*.npz)."""

from functools import lru_cache
from pathlib import Path
from types import SimpleNamespace

import numpy as np

from paper_2506_23568_b200.model import (DataCube, FrequencyGrid, ImagingRegion,
                                         SyntheticAperture)

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def load_npz(name: str) -> dict:
    """The raw arrays of a golden file (cases without an aperture/cube)."""
    return dict(np.load(GOLDEN / f"{name}.npz"))


def load(name: str) -> SimpleNamespace:
    z = dict(np.load(GOLDEN / f"{name}.npz"))
    f = z["freqs"]
    freqs = FrequencyGrid(float(f[0]), float(f[1]), int(f[2]))
    nx, ny = (int(v) for v in z["nxny"])
    ap = SyntheticAperture(elements=z["elements"], nx=nx, ny=ny)
    region = ImagingRegion(*(float(v) for v in z["region"]))
    cube = DataCube(values=z["cube"], aperture=ap, freqs=freqs)
    return SimpleNamespace(z=z, freqs=freqs, aperture=ap, region=region, cube=cube,
                           dims=tuple(int(d) for d in z["dims"]))


def provenance(z: dict, prefix: str) -> dict:
    sizes = z[prefix + "_level_sizes"]
    flat = z[prefix + "_level_points"].tolist()
    lp, i = [], 0
    for s in sizes:
        lp.append(flat[i:i + s])
        i += s
    return {"level_points": lp, "merge_flags": z[prefix + "_merge_flags"].tolist(),
            "final_flags": int(z[prefix + "_final_flags"])}


def grid_valid(z: dict, prefix: str) -> list:
    dims = z[prefix + "_dims"]
    n = int(np.prod(dims, axis=1).sum())
    bits = np.unpackbits(z[prefix + "_valid"])[:n].astype(bool)
    out, i = [], 0
    for d in dims:
        k = int(np.prod(d))
        out.append(bits[i:i + k].reshape(tuple(d)))
        i += k
    return out


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))
