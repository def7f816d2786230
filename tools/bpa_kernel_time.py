"""Median device time of the config-1 BPA kernel call (hhsar_bpa_cartesian);
HHSAR_LIB=<other build> A/Bs another library build in a separate process."""
import os
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2506_23568_b200 import _native, bpa, rangecomp, workloads
    w = workloads.config(int(os.environ.get("CFG", "1")))
    cube = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                            w.freqs.k_samples)
    el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
    el4 = bpa.el_f32x4(el)
    env, dt, k_ref = rangecomp.range_compress_device(cube, w.freqs, w.upsample)
    out = torch.empty(w.n_voxels, dtype=torch.complex64, device="cuda")
    times = []
    for i in range(6):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        bpa.bpa_volume_device(env, el4, w.region, w.dims, 0.0, dt, k_ref, out=out)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    ms = statistics.median(times[1:])
    print(f"lib {os.environ.get('HHSAR_LIB', 'default')}: {ms:.3f} ms, "
          f"{w.bpa_units / ms / 1e6:.1f} Gunit/s")
    np.save(f"/tmp/bpa_out_{Path(os.environ.get('HHSAR_LIB', 'default')).stem}.npy", out.cpu().numpy())


if __name__ == "__main__":
    main()
