import ctypes, statistics, torch
from pathlib import Path
lib = ctypes.CDLL(str(Path(__file__).with_name("_bw.so")))
n_el, n_f = 2097152, 1024
cube = torch.randn((n_el, n_f), dtype=torch.complex64, device="cuda")
out = torch.empty((n_el, 4 * n_f), dtype=torch.complex64, device="cuda")
ts = []
for _ in range(6):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); lib.bw_rw14(ctypes.c_void_p(cube.data_ptr()), ctypes.c_void_p(out.data_ptr()), ctypes.c_int64(n_el), n_f); e.record()
    torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
ms = statistics.median(ts[1:])
print(f"read 1 : write 4 streaming, no math: {ms:.2f} ms, {(cube.numel() + out.numel()) * 8 / ms / 1e6:.0f} GB/s")
