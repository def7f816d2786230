"""Per-leaf delay span actually read by the leaf stage (config 4 by default):
for every leaf grid, the triangle-inequality window the leaf kernel stages
from -- [min |p - c| - r_e, max |p - c| + r_e] over its VALID lattice points
p (c = element-box centre, r_e = max element distance from c) -- in profile
bins, against the global range gate.  Decides whether per-leaf range gating
would shrink the compressed window."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2506_23568_b200 import ffbp, rangecomp, workloads
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    w = workloads.config(cfg)
    el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
    params = ffbp.FfbpParams(levels=w.levels)
    sched = ffbp.Schedule.shared(w.n_elements, w.levels, w.merge_factor)
    n_t, dt, k_ref, _ = rangecomp.profile_axis(w.freqs, w.upsample)
    lat = ffbp.build_lattices(el, sched, w.region, w.freqs, params.gamma, params.margin,
                              ffbp.src_pad_of(params), (n_t - 1) * dt, gate_dt=dt,
                              gate_bins=n_t)
    torch.cuda.synchronize()
    inv_bin = 2.0 / (ffbp.C_LIGHT * dt)
    a, b = sched.level_slices[0]
    d = lat.descs
    spans, lo_b, hi_b = [], [], []
    for g in range(a, b):
        off, npts = int(d["offset"][g]), int(lat.npts[g])
        v = lat.valid[off:off + npts].bool()
        p = lat.positions[off:off + npts][v]
        s, e = int(d["start"][g]), int(d["stop"][g])
        els = el[s:e]
        c = 0.5 * (els.min(0).values + els.max(0).values)
        re = float((els - c).norm(dim=1).max())
        r = (p - c).norm(dim=1)
        lo = float(r.min()) - re
        hi = float(r.max()) + re
        lo_b.append(lo * inv_bin)
        hi_b.append(hi * inv_bin)
        spans.append((hi - lo) * inv_bin)
    spans = np.array(spans)
    lo_b, hi_b = np.array(lo_b), np.array(hi_b)
    print(f"config {cfg}: {len(spans)} leaves, global gate {lat.gate}, n_t {n_t}")
    print(f"valid-point span (bins, before pad): min {spans.min():.1f} median "
          f"{np.median(spans):.1f} p90 {np.percentile(spans, 90):.1f} max {spans.max():.1f}")
    print(f"union over leaves: [{lo_b.min():.1f}, {hi_b.max():.1f}] = {hi_b.max() - lo_b.min():.1f} bins")


if __name__ == "__main__":
    main()
