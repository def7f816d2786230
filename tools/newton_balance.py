"""Newton work balance: per grid level, active columns, planes per column and
Newton iterations per column (config 3 by default)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import bpa, ffbp, workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = workloads.config(cfg)
gen = torch.Generator(device="cuda").manual_seed(w.seed)
cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda", generator=gen)
el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
el4 = bpa.el_f32x4(el)
run = ffbp.hhffbpa_from_cube(cube, el, el4, w.freqs, w.region, w.dims,
                             ffbp.FfbpParams(levels=w.levels), w.levels, w.merge_factor, w.upsample)
torch.cuda.synchronize()
d = run.lattices.descs
st = run.lattices.stats.cpu().numpy()
span = np.maximum(d["act_hi"].astype(np.int64) - d["act_lo"] + 1, 0)
cols = span[:, 0] * span[:, 1]
planes = d["near_hi"][:, 2].astype(np.int64) + 1
for k, (a, b) in enumerate(run.sched.level_slices):
    c = cols[a:b].sum()
    it = st[a:b, 4].sum()
    print(f"level {k}: grids {b - a:5d} columns {c:8d} planes/col {planes[a:b].mean():6.1f} "
          f"(max {planes[a:b].max()}) iterations {it:10d} it/col {it / max(c, 1):7.1f} "
          f"it/solve {it / max(st[a:b, 5].sum(), 1):5.2f}")
print("total columns", cols.sum(), "iterations", st[:, 4].sum())
