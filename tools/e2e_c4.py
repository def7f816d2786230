"""Where the config-4 end-to-end call (public hhffbpa_reconstruct from a
pinned host cube) spends its time: the call's phases with a device sync
after each, plus the pinned H2D / D2H rates of this box."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2506_23568_b200 as hh  # noqa: E402
from paper_2506_23568_b200 import _native, bpa, ffbp, workloads  # noqa: E402
from paper_2506_23568_b200.bpa import _finish, region_grid  # noqa: E402
from paper_2506_23568_b200.model import DataCube  # noqa: E402
from paper_2506_23568_b200.rangecomp import CubeUpload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = workloads.config(cfg)
el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
cube_dev = _native.simulate_uniform(el, w.scene_pos, w.scene_refl, w.freqs)
host = torch.empty(cube_dev.shape, dtype=torch.complex64, pin_memory=True)
host.copy_(cube_dev)
del cube_dev
torch.cuda.synchronize()
data = DataCube(values=host.numpy(), aperture=w.aperture, freqs=w.freqs)
params = ffbp.FfbpParams(levels=w.levels)
for _ in range(2):
    hh.hhffbpa_reconstruct(data, w.region, w.dims, params, upsample=w.upsample,
                           merge_factor=w.merge_factor)
torch.cuda.synchronize()
t = time.perf_counter()
hh.hhffbpa_reconstruct(data, w.region, w.dims, params, upsample=w.upsample,
                       merge_factor=w.merge_factor)
print(f"{(time.perf_counter() - t) * 1e3:8.1f} ms  full call")

marks = [("start", time.perf_counter())]


def mark(name, sync=True):
    if sync:
        torch.cuda.synchronize()
    marks.append((name, time.perf_counter()))


el_dev = torch.tensor(np.ascontiguousarray(w.aperture.elements, dtype=np.float64), device="cuda")
mark("elements H2D")
ups = []


def factory():
    mark("plan queued (upload starts)", sync=False)
    ups.append(CubeUpload(data.values))
    return ups[0]


ffbp._trace = lambda label: mark(f"  trace: {label}", sync=False)
run = ffbp.hhffbpa_from_cube(None, el_dev, bpa.el_f32x4(el_dev), w.freqs, w.region, w.dims,
                             params, w.levels, w.merge_factor, w.upsample, upload=factory)
ffbp._trace = None
mark("hhffbpa_from_cube enqueue", sync=False)
ev = torch.cuda.Event()
ev.record()
for _, _, e in ups[0].chunks[-1:]:
    e.synchronize()
mark("last cube chunk landed", sync=False)
torch.cuda.synchronize()
mark("device done (upload + step)")
origin, step = region_grid(w.region, w.dims)
extra = torch.cat([run.flags, run.lattices.stats.reshape(-1)])
vol, _ = _finish(run.volume, run.oow, w.dims, origin, step, {}, extra)
mark("_finish (checks, D2H volume)")
prev = marks[0][1]
for name, tm in marks[1:]:
    print(f"{(tm - prev) * 1e3:8.1f} ms  {name}")
    prev = tm
n = host.numel() * 8
for label, fn in (("H2D pinned", lambda d: d.copy_(host, non_blocking=True)),):
    d = torch.empty_like(host, device="cuda")
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn(d)
    torch.cuda.synchronize()
    s = time.perf_counter() - t
    print(f"{label}: {n / s / 1e9:.1f} GB/s ({s * 1e3:.1f} ms for {n / 1e9:.1f} GB)")
v = run.volume
hv = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
torch.cuda.synchronize()
t = time.perf_counter()
hv.copy_(v, non_blocking=True)
torch.cuda.synchronize()
s = time.perf_counter() - t
print(f"D2H pinned: {v.numel() * 8 / s / 1e9:.1f} GB/s ({s * 1e3:.1f} ms)")

import cProfile  # noqa: E402
import pstats  # noqa: E402

pr = cProfile.Profile()
torch.cuda.synchronize()
pr.enable()
hh.hhffbpa_reconstruct(data, w.region, w.dims, params, upsample=w.upsample,
                       merge_factor=w.merge_factor)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
