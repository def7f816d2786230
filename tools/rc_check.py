"""Fused range compression vs the cuFFT path: accuracy and device time."""
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import _native, rangecomp, workloads  # noqa: E402

for cfg in (0, 1, 3):
    w = workloads.config(cfg)
    cube = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                            w.freqs.k_samples)

    def timed(force):
        rangecomp._FORCE_CUFFT = force
        ts = []
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            p, dt, kr = rangecomp.range_compress_device(cube, w.freqs, w.upsample)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        return p, statistics.median(ts[1:])

    a, ta = timed(False)
    b, tb = timed(True)
    err = (torch.linalg.norm(a - b) / torch.linalg.norm(b)).item()
    nbytes = cube.numel() * 8 + a.numel() * 8
    print(f"config {cfg}: fused {ta:.3f} ms ({nbytes / ta / 1e6:.0f} GB/s) vs cufft+demod "
          f"{tb:.3f} ms, rel diff {err:.2e}")
