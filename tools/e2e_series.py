import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, "/root/repo")
import torch
from paper_2506_23568_b200 import _native, bpa, workloads
from paper_2506_23568_b200.model import DataCube
w = workloads.config(1)
cube_dev = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl, w.freqs.k_samples)
host = cube_dev.cpu().pin_memory()
cube = DataCube(values=host.numpy(), aperture=w.aperture, freqs=w.freqs)
for i in range(12):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = bpa.bpa_reconstruct(cube, w.region, dims=w.dims, upsample=w.upsample)
    torch.cuda.synchronize()
    print(f"{i}: {1e3 * (time.perf_counter() - t):.2f} ms")
