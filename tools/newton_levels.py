"""Newton iterations / solves / valid points per tree level of a BASELINE
config (which grids the inversion work sits in)."""
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
    n_t, dt, _, _ = rangecomp.profile_axis(w.freqs, w.upsample)
    lat = ffbp.build_lattices(el, sched, w.region, w.freqs, params.gamma, params.margin,
                              ffbp.src_pad_of(params), (n_t - 1) * dt)
    torch.cuda.synchronize()
    st = lat.stats.cpu().numpy()
    tot = st[:, 4].sum()
    for k, (a, b) in enumerate(sched.level_slices):
        it = int(st[a:b, 4].sum())
        print(f"config {cfg} grid level {k}: {b - a} grids, {lat.npts[a:b].sum()} lattice points, "
              f"{int(st[a:b, 0].sum())} valid, {int(st[a:b, 5].sum())} solves, {it} iterations "
              f"({it / tot:.1%})")


if __name__ == "__main__":
    main()
