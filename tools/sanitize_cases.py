"""Small cases of every CUDA entry point of the library, meant for
compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py

(the GPU pool this build ran on refuses compute-sanitizer, so in round 2
the cases ran plain, every result checked by the GPU parity tests instead).

HHFFBPA (binary and factor 4, linear and cubic, range-gated: the leaf
kernel's staging, Newton's heavy / light / fix-up phases, merges, the
Cartesian landing -- series and per-voxel), direct BPA (tile and gather
kernels), the windowed range compression at both split-kernel row lengths
and the Stockham / cuFFT paths, the Born simulators, psnr / MIP, and the
operator-level entry points."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2506_23568_b200 as hh
    from paper_2506_23568_b200 import _native, bpa, ffbp, rangecomp, workloads
    from paper_2506_23568_b200.model import FrequencyGrid
    w = workloads.config(2, frames=64)
    cube = workloads.simulate_numpy(w)
    dims = (24, 24, 12)
    for mf, kernel, levels in ((2, "linear", 4), (4, "linear", 5), (4, "cubic", 5)):
        v = hh.hhffbpa_reconstruct(cube, w.region, dims, hh.FfbpParams(levels=levels,
                                                                       kernel=kernel),
                                   upsample=4, merge_factor=mf)
        print(f"hhffbpa factor {mf} {kernel}: |v| {np.abs(v.values).max():.3e}", flush=True)
    ffbp.LANDING_SERIES, ffbp.LANDING_PAIRS = False, False  # per-voxel landing, direct gathers
    v2 = hh.hhffbpa_reconstruct(cube, w.region, dims, hh.FfbpParams(levels=4), upsample=4)
    ffbp.LANDING_SERIES, ffbp.LANDING_PAIRS = True, True
    b = hh.bpa_reconstruct(cube, w.region, dims=dims, upsample=4)
    print(f"bpa: |v| {np.abs(b.values).max():.3e}, psnr {hh.psnr(b, v2):.1f} dB", flush=True)
    mip = hh.max_intensity_projection(b, "z")
    pts = np.random.default_rng(0).uniform(-0.02, 0.02, (100, 3)) + np.array([0, 0, 0.3])
    prof = hh.range_compress(cube, upsample=4)
    g = hh.backproject(prof, slice(0, 64), pts)
    print(f"gather: {np.abs(g).max():.3e}, mip {mip.max():.3f}", flush=True)
    for n_el, n_f, up, b0, width in ((70, 1024, 4, 65, 128), (70, 1024, 4, 1, 255),
                                     (70, 512, 4, 10, 64), (33, 256, 4, 5, 100),
                                     (9, 300, 4, 0, 1200)):
        freqs = FrequencyGrid(77e9, 81e9, n_f)
        c = torch.randn((n_el, n_f), dtype=torch.complex64, device="cuda")
        full, _, _ = rangecomp.range_compress_device(c, freqs, up)
        win, *_ = rangecomp.range_compress_window(c, freqs, up, b0, min(width, full.shape[1] - b0))
        torch.cuda.synchronize()
        print(f"range compression {n_el}x{n_f} -> {full.shape[1]} window {win.shape}", flush=True)
    el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
    sim = _native.simulate_uniform(el, w.scene_pos, w.scene_refl, w.freqs)
    torch.cuda.synchronize()
    print(f"simulate_uniform {tuple(sim.shape)}", flush=True)
    print("sanitize cases done", flush=True)


if __name__ == "__main__":
    main()
