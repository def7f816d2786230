"""A/B device time of the fused range compression (full rows and the
HHFFBPA gate) through the C ABI: pre-allocated output, back-to-back launches
between two events (set HHSAR_LIB to time another build)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import _native, rangecomp, workloads  # noqa: E402

GATES = {3: (10, 64), 4: (65, 128), 1: (0, 1024)}
for cfg in [int(c) for c in (sys.argv[1:] or ["1", "3", "4"])]:
    w = workloads.config(cfg)
    gen = torch.Generator(device="cuda").manual_seed(1)
    cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda",
                       generator=gen)
    n_t, dt, k_ref, a = rangecomp.profile_axis(w.freqs, w.upsample)
    res = {}
    for label, (b0, width) in (("full", (0, n_t)), ("gated", GATES[cfg])):
        if label == "full" and cfg == 4 and not hasattr(_native.library(), "hhsar_range_compress_window"):
            pass
        out = torch.empty((w.n_elements, width), dtype=torch.complex64, device="cuda")
        lib = _native.library()
        win = getattr(lib, "hhsar_range_compress_window", None)

        def launch():
            if win is not None:
                _native.call("hhsar_range_compress_window", _native.ptr(cube), w.n_elements,
                             w.freqs.count, n_t, a, dt, b0, width, _native.ptr(out),
                             _native.stream_handle())
            else:
                _native.call("hhsar_range_compress", _native.ptr(cube), w.n_elements,
                             w.freqs.count, n_t, a, dt, _native.ptr(out), _native.stream_handle())
        if win is None and label == "gated":
            continue
        reps = 20 if cfg != 4 else 5
        for _ in range(2):
            launch()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            launch()
        e.record()
        torch.cuda.synchronize()
        res[label] = round(s.elapsed_time(e) / reps, 4)
        del out
        torch.cuda.empty_cache()
    print(f"config {cfg}: {res}", flush=True)
    del cube
    torch.cuda.empty_cache()
