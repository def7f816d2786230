"""cProfile of the host side of hhffbpa_from_cube (config 3 by default)."""
import cProfile
import pstats
import sys
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


def step():
    return ffbp.hhffbpa_from_cube(cube, el, el4, w.freqs, w.region, w.dims, params, w.levels, 2,
                                  w.upsample)


for _ in range(3):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
