"""One warm-up + one HHFFBPA step (hhffbpa_from_cube, seeded random cube) of a
BASELINE config, for ncu captures of single kernels (-k regex:...)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import bpa, ffbp, workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = workloads.config(cfg)
gen = torch.Generator(device="cuda").manual_seed(w.seed)
cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda",
                   generator=gen)
el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
el4 = bpa.el_f32x4(el)
params = ffbp.FfbpParams(levels=w.levels)
for _ in range(2):
    run = ffbp.hhffbpa_from_cube(cube, el, el4, w.freqs, w.region, w.dims, params, w.levels,
                                 w.merge_factor, w.upsample)
torch.cuda.synchronize()
print("done")
