"""Range-gated compression at config 4 (seeded random cube, the gate the
HHFFBPA step uses there) for ncu / timing."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import rangecomp, workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
b0, w_bins = (49, 288) if cfg == 4 else (0, 352)
w = workloads.config(cfg)
gen = torch.Generator(device="cuda").manual_seed(1)
cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda",
                   generator=gen)
ts = []
for _ in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    prof, t0, dt, k_ref = rangecomp.range_compress_window(cube, w.freqs, w.upsample, b0, w_bins)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
print("ms", [round(t, 3) for t in ts])
