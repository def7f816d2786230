"""GPU timeline of one hhffbpa_from_cube step: every native call bracketed
by CUDA events on its own stream, reported relative to a start event on the
caller's stream (config 3 by default, seeded random cube)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import _native, bpa, ffbp, workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = workloads.config(cfg)
gen = torch.Generator(device="cuda").manual_seed(w.seed)
cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda", generator=gen)
el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
el4 = bpa.el_f32x4(el)
params = ffbp.FfbpParams(levels=w.levels)


def step():
    return ffbp.hhffbpa_from_cube(cube, el, el4, w.freqs, w.region, w.dims, params, w.levels,
                                  w.merge_factor, w.upsample)


for _ in range(3):
    step()
torch.cuda.synchronize()
orig = _native.call
log = []


def traced(name, *a):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    orig(name, *a)
    e.record()
    log.append((name, torch.cuda.current_stream().stream_id, s, e))


t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
_native.call = traced
t0.record()
run = step()
t1.record()
torch.cuda.synchronize()
_native.call = orig
print(f"step {t0.elapsed_time(t1):.3f} ms")
for name, sid, s, e in log:
    print(f"  stream {sid:>3}  {t0.elapsed_time(s):7.3f} .. {t0.elapsed_time(e):7.3f} ms  {name}")
