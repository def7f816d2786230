"""Short driver for ncu captures: one warm-up and one profiled step of a
workload (default: BASELINE config 1 direct BPA)."""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--frames", type=int, default=None)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--random", action="store_true", help="seeded random cube (no Born sum)")
    args = ap.parse_args()
    import torch
    from paper_2506_23568_b200 import _native, bpa, ffbp, rangecomp, workloads
    w = workloads.config(args.config, frames=args.frames)
    if args.random:
        gen = torch.Generator(device="cuda").manual_seed(w.seed)
        cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda",
                           generator=gen)
    else:
        cube = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                                w.freqs.k_samples)
    el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
    el4 = bpa.el_f32x4(el)
    for _ in range(args.steps):
        env, dt, k_ref = rangecomp.range_compress_device(cube, w.freqs, w.upsample)
        if w.algorithm == "bpa":
            bpa.bpa_volume_device(env, el4, w.region, w.dims, 0.0, dt, k_ref)
        else:
            ffbp.hhffbpa_device(env, el, el4, 0.0, dt, k_ref, w.freqs, w.region, w.dims,
                                ffbp.FfbpParams(levels=w.levels), w.levels, w.merge_factor)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
