"""A/B of the Cartesian landing: one config's HHFFBPA step (seeded Born
cube) timed as a CUDA-graph replay, and the volume saved to OUT.npy for a
cross-build comparison (set HHSAR_LIB for the other build).
Usage: landing_ab.py CONFIG OUT [compare.npy]"""
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import _native, bpa, ffbp, workloads  # noqa: E402

cfg, out = int(sys.argv[1]), sys.argv[2]
w = workloads.config(cfg)
el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
cube = _native.simulate_uniform(el, w.scene_pos, w.scene_refl, w.freqs)
el4 = bpa.el_f32x4(el)
params = ffbp.FfbpParams(levels=w.levels)
args = (el, el4, w.freqs, w.region, w.dims, params, w.levels, w.merge_factor, w.upsample)
g = ffbp.StepGraph(cube, *args)
ts = []
for it in range(12):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    run = g.replay()
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
vol = run.volume.cpu().numpy()
np.save(out, vol)
msg = f"config {cfg}: step {statistics.median(ts[2:]):.3f} ms"
msg += f", final flags {[int(f) for f in run.flags.cpu().numpy()][-1]}"
if len(sys.argv) > 3:
    ref = np.load(sys.argv[3])
    rel = np.linalg.norm(vol - ref) / np.linalg.norm(ref)
    msg += f", rel-L2 vs {sys.argv[3]}: {rel:.3e}, peak equal {np.argmax(np.abs(vol)) == np.argmax(np.abs(ref))}"
print(msg, flush=True)
