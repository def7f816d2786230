"""The 4096-bin gated range compression against a float64 numpy reference
(rangecomp.py:61-101: zero-pad, unnormalised IFFT, demodulation)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import rangecomp  # noqa: E402
from paper_2506_23568_b200.model import FrequencyGrid  # noqa: E402

for n_f, up, b0, w in [(1024, 4, 49, 288), (1024, 4, 0, 512), (512, 8, 3000, 400), (1024, 4, 4095, 1)]:
    freqs = FrequencyGrid(77e9, 81e9, n_f)
    gen = torch.Generator(device="cuda").manual_seed(n_f + b0)
    cube = torch.randn((512, n_f), dtype=torch.complex64, device="cuda", generator=gen)
    got, t0w, dt, k_ref = rangecomp.range_compress_window(cube, freqs, up, b0, w)
    n_t, dt2, _, a = rangecomp.profile_axis(freqs, up)
    x = cube.cpu().numpy().astype(np.complex128)
    pad = np.zeros((x.shape[0], n_t), complex)
    pad[:, :n_f] = x
    full = np.fft.ifft(pad, axis=1) * n_t * np.exp(1j * a * (dt2 * np.arange(n_t)))
    want = full[:, b0:b0 + w]
    g = got.cpu().numpy()
    rel = np.linalg.norm(g - want) / np.linalg.norm(want)
    mx = np.max(np.abs(g - want)) / np.sqrt(np.mean(np.abs(want) ** 2))
    print(f"n_f {n_f} up {up} gate ({b0},{w}): rel-L2 {rel:.2e} max/rms {mx:.2e}")
