"""Co-residency probe (config 4): the gated range compression (FP32 pipe)
and the leaf stage (SFU pipe), each alone, back to back, and launched
together on two streams (the leaf stage reads an earlier compression's
profiles, so the two are independent here).  If the concurrent pair beats
the back-to-back pair, pipelining the compression with the leaf stage
(rows of leaf group c+1 beside the leaves of group c) would pay.
argv: leaf stream priority (-1 high / 0 normal), optionally 'leaf_first'."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2506_23568_b200 import _native, bpa, ffbp, rangecomp, workloads
    prio = int(sys.argv[1]) if len(sys.argv) > 1 else -1
    leaf_first = "leaf_first" in sys.argv
    w = workloads.config(4)
    el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
    el4 = bpa.el_f32x4(el)
    gen = torch.Generator(device="cuda").manual_seed(1)
    cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda",
                       generator=gen)
    params = ffbp.FfbpParams(levels=w.levels)
    run = ffbp.hhffbpa_from_cube(cube, el, el4, w.freqs, w.region, w.dims, params, w.levels,
                                 w.merge_factor, w.upsample)
    torch.cuda.synchronize()
    b0, gw = run.lattices.gate
    env, t0, dt, k_ref = rangecomp.range_compress_window(cube, w.freqs, w.upsample, b0, gw)
    n_t = w.freqs.count * w.upsample
    pipe = ffbp.Pipeline(env, el, el4, t0, dt, k_ref, w.freqs, w.region, w.dims, params,
                         w.levels, w.merge_factor, window_hi=(n_t - 1) * dt, sched=run.sched,
                         lat=run.lattices)
    main_s = torch.cuda.current_stream()
    side = torch.cuda.Stream(priority=prio)

    def rc():
        rangecomp.range_compress_window(cube, w.freqs, w.upsample, b0, gw)

    def leaf():
        pipe.leaves()

    def timed(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    def both():
        side.wait_stream(main_s)
        if leaf_first:
            with torch.cuda.stream(side):
                leaf()
            rc()
        else:
            rc()
            with torch.cuda.stream(side):
                leaf()
        main_s.wait_stream(side)

    out = {"leaf_priority": prio, "leaf_first": leaf_first}
    out["rc_ms"] = round(timed(rc), 3)
    out["leaf_ms"] = round(timed(leaf), 3)
    out["serial_ms"] = round(timed(lambda: (rc(), leaf())), 3)
    out["concurrent_ms"] = round(timed(both), 3)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
