"""Projected multi-GPU scaling of the sharded HHFFBPA (dist.hhffbpa_sharded_device)
and the voxel-sharded BPA, measured one rank at a time on the single GPU this
build has.  PROJECTION, not a multi-GPU measurement: each rank's pipeline runs
alone (collectives replaced by a counting no-op, so its device time is its
compute share); the exchange is costed from the bytes it would move at a
stated NVLink bandwidth.  Projected time at world W = max over ranks of the
rank's device time + exchange bytes / bandwidth.

    python tools/projected_scaling.py 3 2 4 8     (config, worlds...)
    OUTPUT=all|root|shard python tools/projected_scaling.py 4 2 4 8
      (volume output mode of dist.hhffbpa_sharded_device; default shard,
      the bench's N > 1 mode; CACHED=0: no per-rank plan cache; SPLIT_TOP=1:
      the top grids' Newton split by u-rows across ranks + one all-reduce)
"""
import os
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_23568_b200 import dist, ffbp, workloads  # noqa: E402

NVLINK_GBS = 900.0  # B200 NVLink 5, per direction per GPU


class CountingComm:
    """Collectives as no-ops that count the bytes a ring would move per rank."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world
        self.bytes = 0

    def allreduce_sum(self, t):
        self.bytes += 2 * t.numel() * t.element_size() * (self.world - 1) // self.world

    def allgather_segments(self, buf, segments):
        longest = max(b - a for a, b in segments)
        self.bytes += longest * buf.element_size() * (self.world - 1)

    def gather_segments(self, buf, segments, root=0, base=0):
        # the root receives W-1 segments; the others send one
        longest = max(b - a for a, b in segments)
        self.bytes += longest * buf.element_size() * ((self.world - 1) if self.rank == root else 1)


OUTPUT = os.environ.get("OUTPUT", "shard")
CACHED = os.environ.get("CACHED", "1") == "1"  # per-rank plan cache (the bench's N > 1 step)
SPLIT_TOP = os.environ.get("SPLIT_TOP", "0") == "1"


def time_rank(w, cube, el, params, factor, world, rank, reps=3):
    sched, kx, owned, (e0, e1) = dist.plan_shard(w.n_elements, w.levels, factor, world, rank)
    rows = cube[e0:e1].contiguous()
    best, comm, plan = None, None, None
    for it in range(reps + 1):
        comm = CountingComm(rank, world)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        # as the bench's N-rank step: the first call's plan is cached
        r = dist.hhffbpa_sharded_device(comm, rows, e0, el, w.freqs, w.region, w.dims, params,
                                        w.levels, factor, w.upsample, output=OUTPUT,
                                        plan_cache=plan if CACHED else None,
                                        split_top=SPLIT_TOP)
        plan = r.plan
        e.record()
        torch.cuda.synchronize()
        t = s.elapsed_time(e)
        if it:
            best = t if best is None else min(best, t)
    return best, comm.bytes


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    worlds = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
    w = workloads.config(cfg)
    factor = w.merge_factor
    gen = torch.Generator(device="cuda").manual_seed(w.seed)
    cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda",
                       generator=gen)
    el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
    params = ffbp.FfbpParams(levels=w.levels)
    t1, _ = time_rank(w, cube, el, params, factor, 1, 0)
    out = {"config": cfg, "merge_factor": factor, "one_gpu_ms": round(t1, 3),
           "nvlink_gbs_assumed": NVLINK_GBS, "output": OUTPUT, "split_top": SPLIT_TOP, "note": "projection: ranks timed one at a time "
           "on one B200, collectives costed from bytes", "worlds": {}}
    for W in worlds:
        per = [time_rank(w, cube, el, params, factor, W, r) for r in range(W)]
        ms = [p[0] for p in per]
        comm_ms = max(p[1] for p in per) / (NVLINK_GBS * 1e9) * 1e3
        proj = max(ms) + comm_ms
        out["worlds"][W] = {"rank_ms": [round(x, 3) for x in ms], "exchange_ms": round(comm_ms, 3),
                            "projected_ms": round(proj, 3),
                            "projected_speedup": round(t1 / proj, 2),
                            "projected_efficiency": round(t1 / proj / W, 3)}
        print(json.dumps({W: out["worlds"][W]}), flush=True)
    print(json.dumps(out))




def rank_timeline(cfg=3, world=8, rank=0):
    """Per-call device timeline of one rank's share (where the time goes)."""
    from paper_2506_23568_b200 import _native
    w = workloads.config(cfg)
    gen = torch.Generator(device="cuda").manual_seed(w.seed)
    cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda",
                       generator=gen)
    el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
    params = ffbp.FfbpParams(levels=w.levels)
    time_rank(w, cube, el, params, w.merge_factor, world, rank, reps=1)
    sched, kx, owned, (e0, e1) = dist.plan_shard(w.n_elements, w.levels, w.merge_factor, world,
                                                 rank)
    orig, log = _native.call, []

    def traced(name, *a):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        orig(name, *a)
        e.record()
        log.append((name, s, e))

    t0 = torch.cuda.Event(enable_timing=True)
    _native.call = traced
    t0.record()
    dist.hhffbpa_sharded_device(CountingComm(rank, world), cube[e0:e1].contiguous(), e0, el,
                                w.freqs, w.region, w.dims, params, w.levels, w.merge_factor,
                                w.upsample)
    torch.cuda.synchronize()
    _native.call = orig
    print(f"exchange level {kx}, owned leaves {owned[0]}")
    for name, s, e in log:
        print(f"  {t0.elapsed_time(s):7.3f} .. {t0.elapsed_time(e):7.3f} ms  {name}")


if __name__ == "__main__":
    if sys.argv[1:2] == ["timeline"]:
        rank_timeline(int(sys.argv[2]), int(sys.argv[3]))
    else:
        main()
