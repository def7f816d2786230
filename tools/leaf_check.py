"""Leaf kernel check: device time of hhsar_leaf_bp and the number of (CTA,
element) pairs that fell back to the checked global-gather path (the window
width is chosen per CTA inside the kernel)."""
import ctypes
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
lib = _native.library()
lib.hhsar_debug_leaf_checked.restype = ctypes.c_ulonglong
orig = _native.call
for tw in ["auto"]:
    times = []

    def timed(name, *a):
        if name == "hhsar_leaf_bp":
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            orig(name, *a)
            e.record()
            times.append((s, e))
        else:
            orig(name, *a)

    _native.call = timed
    vols = []
    tw_hist = (ctypes.c_ulonglong * 4)()
    for rep in range(3):
        lib.hhsar_debug_leaf_checked()
        lib.hhsar_debug_leaf_tw(tw_hist)
        run = ffbp.hhffbpa_from_cube(cube, el, el4, w.freqs, w.region, w.dims, params, w.levels,
                                     w.merge_factor, w.upsample)
        torch.cuda.synchronize()
        checked = lib.hhsar_debug_leaf_checked()
        lib.hhsar_debug_leaf_tw(tw_hist)
        vols.append(run.volume)
    _native.call = orig
    ms = min(s.elapsed_time(e) for s, e in times)
    a, b = run.sched.level_slices[0]
    d = run.lattices.descs
    m = (d["stop"][a:b] - d["start"][a:b]).astype(np.int64)
    pts = run.lattices.stats[a:b, 2].cpu().numpy()
    print(f"CTAs per window width 32/64/128/256: {list(tw_hist)}; leaves {b - a}, elements "
          f"per leaf {m.mean():.0f}, points per leaf {pts.mean():.0f}")
    print(f"TW {tw}: leaf {ms:.3f} ms, checked pairs {checked}, "
          f"volume norm {torch.linalg.norm(vols[-1]).item():.6e}", flush=True)
