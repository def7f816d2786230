"""Eager step vs StepGraph replay (device time per step, K timed after W
warm-up) for BASELINE configs."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    sys.argv += [] 
    from paper_2506_23568_b200 import _native, bpa, ffbp, workloads
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    for cfg in [int(c) for c in (sys.argv[1:] or ["2", "3", "4"])]:
        w = workloads.config(cfg)
        el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
        cube = _native.simulate_uniform(el, w.scene_pos, w.scene_refl, w.freqs)
        el4 = bpa.el_f32x4(el)
        params = ffbp.FfbpParams(levels=w.levels)
        args = (el, el4, w.freqs, w.region, w.dims, params, w.levels, w.merge_factor, w.upsample)
        eager_ms, per_e, _ = bench._timed_steps(lambda: ffbp.hhffbpa_from_cube(cube, *args),
                                               20, 5)
        g = ffbp.StepGraph(cube, *args)
        graph_ms, per_g, _ = bench._timed_steps(g.replay, 20, 5)
        print(json.dumps({"config": cfg, "eager_ms": round(eager_ms, 3),
                          "graph_ms": round(graph_ms, 3),
                          "eager_median": round(sorted(per_e)[10], 3),
                          "graph_median": round(sorted(per_g)[10], 3)}), flush=True)
        del g, cube
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
