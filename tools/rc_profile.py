"""Fused range compression on configs 3 and 4 (seeded random cubes) for ncu."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import rangecomp, workloads  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["3", "4"])]:
    w = workloads.config(cfg)
    gen = torch.Generator(device="cuda").manual_seed(1)
    cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda",
                       generator=gen)
    for _ in range(2):
        prof, dt, k_ref = rangecomp.range_compress_device(cube, w.freqs, w.upsample)
    torch.cuda.synchronize()
    del prof, cube
    torch.cuda.empty_cache()
print("done")
