"""Host-side timeline of one hhffbpa_from_cube step (config 3 by default)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import _native, bpa, ffbp, workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = workloads.config(cfg)
cube = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                        w.freqs.k_samples)
el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
el4 = bpa.el_f32x4(el)
params = ffbp.FfbpParams(levels=w.levels)
for _ in range(3):
    ffbp.hhffbpa_from_cube(cube, el, el4, w.freqs, w.region, w.dims, params, w.levels, 2,
                           w.upsample)
torch.cuda.synchronize()
orig = _native.call
log = []


def traced(name, *a):
    t = time.perf_counter()
    orig(name, *a)
    log.append((name, t, time.perf_counter()))


_native.call = traced
ffbp._trace = lambda label: log.append((label, time.perf_counter(), time.perf_counter()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
run = ffbp.hhffbpa_from_cube(cube, el, el4, w.freqs, w.region, w.dims, params, w.levels, 2,
                             w.upsample)
t_host = time.perf_counter() - t0
e1.record()
torch.cuda.synchronize()
t_all = time.perf_counter() - t0
print(f"host returns after {t_host * 1e3:.2f} ms; GPU done after {t_all * 1e3:.2f} ms; "
      f"events {e0.elapsed_time(e1):.2f} ms")
for name, a, b in log:
    print(f"  {1e3 * (a - t0):8.3f} .. {1e3 * (b - t0):8.3f} ms  {name}")
