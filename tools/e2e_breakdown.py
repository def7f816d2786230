"""Wall-clock breakdown of one public bpa_reconstruct call (config 1)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import _native, bpa, rangecomp, workloads  # noqa: E402
from paper_2506_23568_b200.model import DataCube  # noqa: E402

w = workloads.config(1)
cube_dev = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                            w.freqs.k_samples)
host = cube_dev.cpu().pin_memory()
cube = DataCube(values=host.numpy(), aperture=w.aperture, freqs=w.freqs)
for _ in range(2):
    bpa.bpa_reconstruct(cube, w.region, dims=w.dims, upsample=4)
torch.cuda.synchronize()
marks = []


def mark(name):
    torch.cuda.synchronize()
    marks.append((name, time.perf_counter()))


t0 = time.perf_counter()
mark("start")
prof = rangecomp.range_compress(cube, 4)
mark("range_compress (H2D cube + el, FFT, demod)")
bpa.check_delay_window(prof, w.region)
mark("check_delay_window")
el4 = bpa.el_f32x4(prof.elements_dev)
mark("el_f32x4")
vol, oow = bpa.bpa_volume_device(prof.envelopes, el4, w.region, w.dims, prof.t0, prof.dt,
                                 prof.k_ref)
mark("bpa kernel")
origin, step = bpa.region_grid(w.region, w.dims)
res = bpa._finish(vol, oow, w.dims, origin, step, {})
mark("_finish (isfinite, D2H, ImageVolume)")
prev = marks[0][1]
for name, t in marks[1:]:
    print(f"{(t - prev) * 1e3:8.2f} ms  {name}")
    prev = t
t = time.perf_counter()
bpa.bpa_reconstruct(cube, w.region, dims=w.dims, upsample=4)
print(f"{(time.perf_counter() - t) * 1e3:8.2f} ms  full bpa_reconstruct")

import cProfile  # noqa: E402
import pstats  # noqa: E402

pr = cProfile.Profile()
pr.enable()
bpa.bpa_reconstruct(cube, w.region, dims=w.dims, upsample=4)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
