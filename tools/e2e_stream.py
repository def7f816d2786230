"""Public API end to end at one BASELINE config: single hhffbpa_reconstruct
calls vs hhffbpa_reconstruct_stream over K cubes (pinned host buffers),
host wall time per volume."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2506_23568_b200 as hh  # noqa: E402
from paper_2506_23568_b200 import _native, ffbp, workloads  # noqa: E402
from paper_2506_23568_b200.model import DataCube  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
k = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = workloads.config(cfg)
el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
cube_dev = _native.simulate_uniform(el, w.scene_pos, w.scene_refl, w.freqs)
host = torch.empty(cube_dev.shape, dtype=torch.complex64, pin_memory=True)
host.copy_(cube_dev)
del cube_dev
torch.cuda.synchronize()
data = DataCube(values=host.numpy(), aperture=w.aperture, freqs=w.freqs)
params = ffbp.FfbpParams(levels=w.levels)
kw = dict(upsample=w.upsample, merge_factor=w.merge_factor)
for _ in range(2):
    v = hh.hhffbpa_reconstruct(data, w.region, w.dims, params, **kw)
del v
t = time.perf_counter()
for _ in range(k):
    v = hh.hhffbpa_reconstruct(data, w.region, w.dims, params, **kw)
single = (time.perf_counter() - t) / k
del v
for _ in range(2):
    for v in ffbp.hhffbpa_reconstruct_stream([data] * 4, w.region, w.dims, params, **kw):
        pass
del v
t = time.perf_counter()
n = 0
stamps = []
for v in ffbp.hhffbpa_reconstruct_stream([data] * k, w.region, w.dims, params, **kw):
    n += 1
    stamps.append(time.perf_counter() - t)
stream = (time.perf_counter() - t) / n
print("yield times (s):", [round(x, 3) for x in stamps])
print(f"config {cfg}: single call {single * 1e3:.1f} ms/volume, stream of {n} "
      f"{stream * 1e3:.1f} ms/volume")
