"""Device time of the Newton inversion alone (hhsar_grid_newton on a planned
schedule; plan excluded) for BASELINE configs: median of 10 launches."""
import json
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2506_23568_b200 import ffbp, rangecomp, workloads
    for cfg in [int(c) for c in (sys.argv[1:] or ["3", "4"])]:
        w = workloads.config(cfg)
        el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
        params = ffbp.FfbpParams(levels=w.levels)
        sched = ffbp.Schedule.shared(w.n_elements, w.levels, w.merge_factor)
        n_t, dt, _, _ = rangecomp.profile_axis(w.freqs, w.upsample)
        ts, iters = [], None
        for _ in range(12):
            pending = ffbp.plan_lattices(el, sched, w.region, w.freqs, params.gamma, params.margin,
                                         ffbp.src_pad_of(params), (n_t - 1) * dt)
            pending["done"].synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            lat = ffbp.finish_lattices(pending)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
            iters = int(lat.stats[:, 4].sum())
        print(json.dumps({"config": cfg, "newton_ms": round(statistics.median(ts[2:]), 3),
                          "iterations": iters}), flush=True)


if __name__ == "__main__":
    main()
