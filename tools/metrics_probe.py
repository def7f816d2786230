"""GPU metrics timing on a config-4-sized volume (1024 x 1024 x 256 complex64)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import metrics  # noqa: E402

v = torch.randn((1024, 1024, 256), dtype=torch.complex64, device="cuda")
t = v * (0.5 + 0.25j)
for f, name in [(lambda: metrics.psnr_device(v, t), "psnr"), (lambda: metrics.mip_device(v, 2), "mip z"),
                (lambda: metrics.mip_device(v, 0), "mip x")]:
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    print(name, round((time.perf_counter() - t0) / 5 * 1e3, 3), "ms", flush=True)
