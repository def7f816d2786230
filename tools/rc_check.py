"""Fused range compression vs the cuFFT path: accuracy and device time."""
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import _native, rangecomp, workloads  # noqa: E402

cfgs = [int(c) for c in (sys.argv[1:] or ["0", "1", "3", "4"])]
for cfg in cfgs:
    w = workloads.config(cfg)
    if cfg == 4:  # no Born simulation at this size: seeded random cube
        gen = torch.Generator(device="cuda").manual_seed(1)
        cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda",
                           generator=gen)
    else:
        cube = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                                w.freqs.k_samples)

    def timed(force):
        rangecomp._FORCE_CUFFT = force
        ts = []
        for it in range(6):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            p, dt, kr = rangecomp.range_compress_device(cube, w.freqs, w.upsample)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
            if it < 5:
                del p
        return p, statistics.median(ts[1:])

    a, ta = timed(False)
    nbytes = cube.numel() * 8 + a.numel() * 8
    msg = f"config {cfg}: fused {ta:.3f} ms ({nbytes / ta / 1e6:.0f} GB/s)"
    if cfg != 4:
        b, tb = timed(True)
        err = (torch.linalg.norm(a - b) / torch.linalg.norm(b)).item()
        msg += f" vs cufft+demod {tb:.3f} ms, rel diff {err:.2e}"
        del b
    else:  # spot-check 64 rows against cuFFT
        sub = cube[:64].contiguous()
        rangecomp._FORCE_CUFFT = True
        b, _, _ = rangecomp.range_compress_device(sub, w.freqs, w.upsample)
        err = (torch.linalg.norm(a[:64] - b) / torch.linalg.norm(b)).item()
        msg += f", rows 0-63 rel diff vs cufft {err:.2e}"
        rangecomp._FORCE_CUFFT = False
    print(msg, flush=True)
    del a, cube
    torch.cuda.empty_cache()
