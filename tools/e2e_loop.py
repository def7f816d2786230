"""e2e call timing: keep vs drop results, and GC effects."""
import gc
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import _native, bpa, workloads  # noqa: E402
from paper_2506_23568_b200.model import DataCube  # noqa: E402

w = workloads.config(1)
cube_dev = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                            w.freqs.k_samples)
host = cube_dev.cpu().pin_memory()
cube = DataCube(values=host.numpy(), aperture=w.aperture, freqs=w.freqs)
for _ in range(2):
    r = bpa.bpa_reconstruct(cube, w.region, dims=w.dims, upsample=4)
for trial in range(3):
    t = time.perf_counter()
    r = bpa.bpa_reconstruct(cube, w.region, dims=w.dims, upsample=4)
    t1 = time.perf_counter()
    del r
    t2 = time.perf_counter()
    print(f"call {1e3 * (t1 - t):.2f} ms, release {1e3 * (t2 - t1):.2f} ms")
gc.disable()
for trial in range(3):
    t = time.perf_counter()
    r = bpa.bpa_reconstruct(cube, w.region, dims=w.dims, upsample=4)
    print(f"gc off: call {1e3 * (time.perf_counter() - t):.2f} ms")
