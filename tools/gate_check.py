"""Range gate: window width per config, gated vs full-profile HHFFBPA
(image difference, oow) and device time of both."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2506_23568_b200 import bpa, ffbp, rangecomp, workloads
    for config in [int(c) for c in (sys.argv[1:] or ["2", "3", "4"])]:
        w = workloads.config(config)
        gen = torch.Generator(device="cuda").manual_seed(w.seed)
        cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda",
                           generator=gen)
        el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
        el4 = bpa.el_f32x4(el)
        params = ffbp.FfbpParams(levels=w.levels)
        out = {"config": config}
        vols = {}
        for gate in (False, True):
            times = []
            for _ in range(5):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                run = ffbp.hhffbpa_from_cube(cube, el, el4, w.freqs, w.region, w.dims, params,
                                             w.levels, w.merge_factor, w.upsample, gate=gate)
                e.record()
                torch.cuda.synchronize()
                times.append(s.elapsed_time(e))
            vols[gate] = run.volume.cpu().numpy()
            out[f"ms_gate_{gate}"] = round(min(times[2:]), 3)
            out[f"oow_gate_{gate}"] = int(run.oow.cpu()[0])
            if gate:
                n_t, dt, _, _ = rangecomp.profile_axis(w.freqs, w.upsample)
                out["gate"] = list(ffbp.leaf_range_gate(run.lattices, run.sched, dt, n_t))
                out["n_t"] = n_t
        out["rel"] = float(np.linalg.norm(vols[True] - vols[False]) / np.linalg.norm(vols[False]))
        print(json.dumps(out), flush=True)
        del cube, run, vols
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
