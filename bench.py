#!/usr/bin/env python
"""Benchmark: BASELINE config 1 -- direct BPA of the handheld MIMO workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric (BASELINE.json): giga voxel x aperture-element backprojections per
second, whole job (all ranks), plus volumes/s.  Workload: 32,000 elements
(4,000 freehand frames x 8 virtual phase centres), 256 frequencies over
77-81 GHz range-compressed to 1,024 bins, 200x200x64 voxels ->
8.192e10 voxel-element units per volume.

One step = range compression (cuFFT + demodulation kernel) + the
hhsar_bpa_cartesian kernel over this rank's voxel slab + (N > 1) the NCCL
all-gather of the slabs.  ``value`` is measured with the cube resident in
HBM; ``e2e`` through the public API (host cube in pinned memory -> H2D ->
reconstruct -> D2H of the complex64 volume).  The profiles (262 MB per step)
exceed the 126 MB L2, so no explicit flush is needed between steps.

``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port of hhsar's Numba loop, oracle/oracle_kernels.c, OpenMP on all
host cores) on a bounded voxel sample of the same workload.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "giga voxel·aperture-element backprojections/s"
UNIT = "Gvoxel·element/s"


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def measured_peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            pass
    return {}


def sfu_peak_units(sm_count: int, mhz: float, mufu_per_unit: int = 3) -> float:
    """SFU ceiling of the BPA unit: 16 MUFU ops / clk / SM (rsqrt + sin + cos
    per unit)."""
    return sm_count * 16 * mhz * 1e6 / mufu_per_unit


def make_workload():
    from paper_2506_23568_b200 import workloads
    return workloads.config(1)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = _dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)

    from paper_2506_23568_b200 import _native, bpa, dist as hdist, rangecomp, workloads
    _native.library()
    w = make_workload()
    n_el, n_vox = w.n_elements, w.n_voxels
    # input cube, generated on the device with the Born simulator (float64 phases)
    cube_dev = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                                w.freqs.k_samples, device=dev)
    torch.cuda.synchronize()
    el_dev = torch.tensor(np.asarray(w.aperture.elements), device=dev)
    el4 = bpa.el_f32x4(el_dev)
    n_t, dt, k_ref, _ = rangecomp.profile_axis(w.freqs, w.upsample)
    vb, ve = hdist.shard_range(n_vox, rank, world)
    chunk = hdist.chunk_size(n_vox, world)
    out = torch.zeros(chunk, dtype=torch.complex64, device=dev)
    full = torch.empty(chunk * world, dtype=torch.complex64, device=dev)
    oow = torch.zeros(1, dtype=torch.int64, device=dev)
    k_start = torch.cuda.Event(enable_timing=True)
    k_end = torch.cuda.Event(enable_timing=True)
    kernel_ms = []

    def step(record_kernel=False):
        env, _, _ = rangecomp.range_compress_device(cube_dev, w.freqs, w.upsample)
        if record_kernel:
            k_start.record()
        bpa.bpa_volume_device(env, el4, w.region, w.dims, 0.0, dt, k_ref, vox_range=(vb, ve),
                              out=out[:ve - vb], oow=oow)
        if record_kernel:
            k_end.record()
        if world > 1:
            dist.all_gather_into_tensor(full, out)
        return env

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index if world > 1 else int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0)) as clocks:
        torch.cuda.synchronize()
        t0.record()
        for _ in range(args.steps):
            step()
        t1.record()
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    # kernel-only timing for the roofline (same stream, separate pass)
    for _ in range(max(1, min(args.steps, 3))):
        step(record_kernel=True)
        torch.cuda.synchronize()
        kernel_ms.append(k_start.elapsed_time(k_end))
    kms = statistics.median(kernel_ms)
    if world > 1:
        t = torch.tensor([ms, kms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kms = float(t[0]), float(t[1])
    if int(oow.cpu()[0]):
        raise RuntimeError("out-of-window delays in the benchmark geometry")

    units = float(n_vox) * n_el
    value = units / (ms / 1e3) / 1e9

    # e2e through the public API with a pinned host cube
    e2e = None
    cube_host = cube_dev.cpu().pin_memory()
    from paper_2506_23568_b200.model import DataCube
    cube = DataCube(values=cube_host.numpy(), aperture=w.aperture, freqs=w.freqs)
    api = (bpa.bpa_reconstruct if world == 1 else
           lambda c, r, dims, upsample: hdist.bpa_reconstruct_sharded(c, r, dims, upsample))
    for _ in range(2):
        vol = api(cube, w.region, dims=w.dims, upsample=w.upsample)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # each call timed on the host clock around the public API (it returns a
    # host volume: the device work is complete); median of the calls
    e2e_steps = max(3, min(args.steps, 5))
    calls = []
    for _ in range(e2e_steps):
        t_e = time.perf_counter()
        vol = api(cube, w.region, dims=w.dims, upsample=w.upsample)
        torch.cuda.synchronize()
        calls.append(time.perf_counter() - t_e)
    e2e_s = statistics.median(calls)
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
    h2d = int(cube_host.numel() * 8 + n_el * 3 * 8)
    d2h = int(n_vox * 8)
    e2e = {"value": round(units / e2e_s / 1e9, 3), "unit": UNIT,
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ms_per_step": round(e2e_s * 1e3, 3), "calls": e2e_steps, "timing": "median call",
           "api": "bpa_reconstruct" if world == 1 else "dist.bpa_reconstruct_sharded"}

    result = None
    if rank == 0:
        peaks = measured_peaks()
        sms = _native.library().hhsar_device_sm_count()
        max_mhz = float(peaks.get("sm_max_mhz", 1965.0))
        csum = clocks.summary()
        shard_units = float(ve - vb) * n_el
        achieved = shard_units / (kms / 1e3) / 1e9
        peak = sfu_peak_units(sms, max_mhz) / 1e9
        hbm_bytes = n_el * n_t * 8 + (ve - vb) * 8
        traffic = None
        try:
            t = json.loads((REPO / "profiles" / "traffic.json").read_text())["bpa_tile_kernel"]
            traffic = int(t["dram_read_bytes"] + t["dram_write_bytes"])
        except Exception:
            pass
        roofline = {
            "kernel": "bpa_tile_kernel (hhsar_bpa_cartesian)", "bound": "sfu",
            "achieved": round(achieved, 2),
            "peak": round(peak, 2), "unit": "Gunit/s", "frac": round(achieved / peak, 4),
            "peak_source": f"{sms} SMs x 16 MUFU/clk x {max_mhz:.0f} MHz / 3 MUFU per unit "
                           "(rsqrt, sin, cos); MEASURED_PEAKS.json has no SFU figure",
            "traffic": traffic,
            "traffic_source": "profiles/traffic.json (ncu --set full, DRAM read+write per launch)",
            "kernel_ms": round(kms, 3),
            "share_of_step": round(kms / ms, 4),
            "hbm": {"achieved_gbs": round(hbm_bytes / (kms / 1e3) / 1e9, 1),
                    "peak_gbs": peaks.get("hbm_gbs", 6542.1),
                    "algorithmic_bytes": int(hbm_bytes)},
        }
        result = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32/c64 (f64 geometry)", "data": "synthetic (seeded Born simulation, GPU)",
            "config": {"workload": "BASELINE config 1: direct BPA, 32,000-element freehand MIMO "
                                   "aperture, 256 freqs -> 1,024 bins, 200x200x64 voxels",
                       "units_per_step": units, "n_elements": n_el, "voxels": list(w.dims),
                       "n_t": n_t, "parallelism": f"voxel-sharded x{world}" if world > 1 else "1 GPU",
                       "l2": "inputs larger than L2 (262 MB profiles per step)"},
            "volumes_per_s": round(1e3 / ms, 3),
            "e2e": e2e, "roofline": roofline, "clocks": csum,
            "gpu_launches": 4 * args.steps,
            "gpu_launches_note": "per step: rc_tables_kernel + range_compress_kernel "
                                 "(hhsar_range_compress) + bpa_tile_kernel + add_parts_kernel "
                                 "(hhsar_bpa_cartesian)",
        }
        # GPU timing legs first; the CPU-heavy legs (oracle parity, CPU
        # baseline) last, so host threads they leave behind cannot perturb
        # the host-orchestrated HHFFBPA steps
        if world == 1 and not args.no_hhffbpa:
            # sub-3 ms steps: 20 timed steps so a rare host hiccup (one step
            # of +0.7..3 ms seen now and then) does not dominate the mean
            result["hhffbpa"] = {f"config{c}": hhffbpa_leg(c, dev, max(args.steps, 20))
                                 for c in (2, 3)}
            free, _ = torch.cuda.mem_get_info(dev)
            if free > 60e9:  # config 4: 17 GB cube + 4.8 GB gated profiles + lattices + volume
                result["hhffbpa"]["config4"] = hhffbpa_leg(4, dev, min(args.steps, 3))
            result["hhffbpa"]["config2_leaf_sweep"] = leaf_sweep_leg(dev, args.steps)
            check = hhffbpa_leg(2, dev, 1, check=True)
            for k in ("parity_vs_oracle", "cpu_oracle_s", "cpu_oracle_cores"):
                result["hhffbpa"]["config2"][k] = check[k]
        if world == 1 and not args.no_cpu_baseline:
            result["cpu_baseline"], result["parity"] = cpu_baseline_leg(w, out[:ve - vb], dt, k_ref)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


def metrics_leg(volume, dims):
    """GPU psnr + max-intensity projection of a device volume (SURVEY
    §8(f) #4): psnr streams both volumes twice (4 x 8 B per voxel), the MIP
    once; reported against the HBM roofline."""
    import torch
    from paper_2506_23568_b200 import metrics
    test = volume * (0.5 + 0.25j)
    n = volume.numel()

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) / reps * 1e3

    ps = timed(lambda: metrics.psnr_device(volume, test))
    mp = timed(lambda: metrics.mip_device(volume.view(*dims), "z"))
    value = metrics.psnr_device(volume, test)
    hbm = measured_peaks().get("hbm_gbs", 6542.1)
    return {"voxels": int(n), "psnr_db": round(value, 3), "psnr_ms": round(ps, 3),
            "psnr_gbs": round(4 * 8 * n / ps / 1e6, 1), "mip_ms": round(mp, 3),
            "mip_gbs": round(8 * n / mp / 1e6, 1), "hbm_peak_gbs": hbm,
            "note": "host wall time per call incl. two scalar read-backs (psnr)"}


def hhffbpa_roofline(w, leaf_units, merge_units, newton_iterations, ms, bins_written=None):
    """SURVEY §8(d)'s path roofline: t_ideal = sum over stages of the time
    the stage's work needs on its bounding unit at B200 peak, frac =
    t_ideal / t_measured (never from BPA-equivalent work)."""
    from paper_2506_23568_b200 import _native
    peaks = measured_peaks()
    sms = _native.library().hhsar_device_sm_count()
    clk = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    hbm = float(peaks.get("hbm_gbs", 6542.1)) * 1e9
    n_t = w.freqs.count * w.upsample
    stages = {
        # bytes: read the cube once, write the envelopes once (only the
        # range-gated bins when the step gates, ffbp.leaf_range_gate)
        "range_compression": w.n_elements * (w.freqs.count + (bins_written or n_t)) * 8 / hbm,
        # ~150 FP64 instructions per iteration (10 sqrt/rsqrt + Jacobian +
        # solve) at 64 lanes / clk / SM (measured 61, tools/bwk/pipes.cu)
        "newton": newton_iterations * 150 / (64 * sms * clk),
        # BPA unit: 3 MUFU at 16 / clk / SM
        "leaf": leaf_units * 3 / (16 * sms * clk),
        # merge unit (point x child): ~45 float64 instructions (4 corner
        # distances, sqrt(r^2 - gap), n, phase) at 64 lanes / clk / SM
        "merges_and_landing": merge_units * 45 / (64 * sms * clk),
    }
    t_ideal = sum(stages.values())
    # the same with the range stage's full-profile bytes (the reference's
    # work: every bin of every envelope), for comparison with ungated runs
    t_full = t_ideal - stages["range_compression"] + w.n_elements * (w.freqs.count + n_t) * 8 / hbm
    return {"t_ideal_ms": round(t_ideal * 1e3, 3), "frac": round(t_ideal * 1e3 / ms, 3),
            "frac_vs_full_profiles": round(t_full * 1e3 / ms, 3),
            "stages_ms": {k: round(v * 1e3, 3) for k, v in stages.items()},
            "method": "SURVEY 8(d): sum over stages of work / bounding-unit peak (HBM "
                      "MEASURED_PEAKS.json; MUFU 16, FP64 64 lanes/clk/SM at the max clock)"}


def leaf_sweep_leg(dev, steps):
    """BASELINE config 2's sweep: HHFFBPA with merge factor 4 and leaves of
    8 / 16 / 32 frames (2^(M-1) balanced leaves of the 4,000 x 8 element
    aperture, M = 10 / 9 / 8), each against direct BPA on the same cube:
    device time per volume, complex rel-L2 and PSNR (GPU metrics) vs BPA."""
    import torch
    from paper_2506_23568_b200 import _native, bpa, ffbp, metrics, rangecomp, workloads
    w = workloads.config(2)
    cube = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                            w.freqs.k_samples, device=dev)
    el = torch.tensor(np.asarray(w.aperture.elements), device=dev)
    el4 = bpa.el_f32x4(el)
    env, dt, k_ref = rangecomp.range_compress_device(cube, w.freqs, w.upsample)
    ref, _ = bpa.bpa_volume_device(env, el4, w.region, w.dims, 0.0, dt, k_ref)
    torch.cuda.synchronize()
    out = {"workload": "BASELINE config 2 sweep: merge factor 4, leaves of 8/16/32 frames "
                       "(M = 10/9/8), accuracy against direct BPA on the same cube"}
    for frames, levels in ((8, 10), (16, 9), (32, 8)):
        params = ffbp.FfbpParams(levels=levels)

        def step():
            return ffbp.hhffbpa_from_cube(cube, el, el4, w.freqs, w.region, w.dims, params,
                                          levels, 4, w.upsample)
        for _ in range(3):
            run = step()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(steps):
            run = step()
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / steps
        v = run.volume
        out[f"leaf_{frames}_frames"] = {
            "levels": levels, "leaf_elements": int(w.n_elements // 2 ** (levels - 1)),
            "ms_per_step": round(ms, 3), "volumes_per_s": round(1e3 / ms, 1),
            "rel_l2_vs_bpa": round((torch.linalg.norm(v - ref) / torch.linalg.norm(ref)).item(), 4),
            "psnr_vs_bpa_db": round(metrics.psnr_device(ref, v), 2)}
    del cube, env, ref
    torch.cuda.empty_cache()
    return out


def hhffbpa_leg(index, dev, steps, check=False):
    """HHFFBPA on BASELINE config `index` (binary schedule, the reference's
    own): device-resident cube, one step = range compression + grids +
    leaf BPA + merges + Cartesian landing.  BPA-equivalent rate =
    N_vox * N_el / t (the unit the paper's speed-up is quoted in)."""
    import torch
    from paper_2506_23568_b200 import _native, bpa, ffbp, rangecomp, workloads
    w = workloads.config(index)
    big = index == 4
    if big:
        # timing and grid statistics are data-independent;
        # the Born sum for 2.1M elements x 1,024 freqs x 20,000 scatterers
        # would take minutes, so a seeded random cube stands in
        gen = torch.Generator(device=dev).manual_seed(w.seed)
        cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device=dev,
                           generator=gen)
    else:
        cube = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                                w.freqs.k_samples, device=dev)
    el = torch.tensor(np.asarray(w.aperture.elements), device=dev)
    el4 = bpa.el_f32x4(el)
    params = ffbp.FfbpParams(levels=w.levels)
    factor = w.merge_factor if big else 2

    def step():
        return ffbp.hhffbpa_from_cube(cube, el, el4, w.freqs, w.region, w.dims, params,
                                      w.levels, factor, w.upsample)

    for _ in range(3):
        run = step()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record()
    for i in range(steps):
        run = step()
        ev[i + 1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[-1]) / steps
    in_order = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    per_step = sorted(in_order)
    stats = run.lattices.stats.cpu().numpy()
    sched, d = run.sched, run.lattices.descs
    g0, g1 = sched.level_slices[0]
    leaf_units = int(sum(int(stats[g, 2]) * int(d["stop"][g] - d["start"][g])
                         for g in range(g0, g1)))
    merge_units = sum(int(stats[a:b, 0].sum()) * f
                      for (a, b), f in zip(sched.level_slices[1:], sched.fanouts))
    merge_units += w.n_voxels * sched.final_children
    sched_name = f"binary M={w.levels}" if factor == 2 else \
        f"merge factor {factor}, M={w.levels}"
    out = {"workload": f"BASELINE config {index}: {w.n_elements} elements, {w.freqs.count} "
                       f"freqs, {list(w.dims)} voxels, {sched_name}"
                       + (", seeded random cube" if big else ""),
           "ms_per_step": round(ms, 3), "volumes_per_s": round(1e3 / ms, 2),
           "step_ms_min_median_max": [round(per_step[0], 3), round(per_step[len(per_step) // 2], 3),
                                      round(per_step[-1], 3)],
           "step_ms": [round(t, 3) for t in in_order],
           "bpa_equivalent_gunits_per_s": round(w.bpa_units / (ms / 1e3) / 1e9, 1),
           "grids": int(sched.n_grids), "leaf_units": leaf_units, "merge_units": merge_units,
           "newton_iterations": int(stats[:, 4].sum()),
           "step": "range compression + grid plan/Newton + leaf BPA + merges + landing"}
    n_t, dt, _, _ = rangecomp.profile_axis(w.freqs, w.upsample)
    gate = ffbp.leaf_range_gate(run.lattices, sched, dt, n_t)
    bins = gate[1]
    out["range_gate"] = {"b0": gate[0], "bins": gate[1], "of": n_t}
    out["roofline"] = hhffbpa_roofline(w, leaf_units, merge_units, int(stats[:, 4].sum()), ms,
                                       bins)
    if check:
        import oracle
        from paper_2506_23568_b200.model import DataCube
        host = DataCube(values=cube.cpu().numpy(), aperture=w.aperture, freqs=w.freqs)
        t = time.perf_counter()
        want, _, _, prov = oracle.hhffbpa_reconstruct(host, w.region, w.dims, levels=w.levels,
                                                      upsample=w.upsample)
        t = time.perf_counter() - t
        got = run.volume.cpu().numpy().reshape(w.dims)
        lp = [[int(v) for v in stats[a:b, 2 if k == 0 else 0]]
              for k, (a, b) in enumerate(sched.level_slices)]
        out["parity_vs_oracle"] = {
            "rel_l2": float(np.linalg.norm(got - want) / np.linalg.norm(want)),
            "peak_index_equal": bool(np.argmax(np.abs(got)) == np.argmax(np.abs(want))),
            "level_points_equal": lp == prov["level_points"][:-1]}
        out["cpu_oracle_s"] = round(t, 2)
        out["cpu_oracle_cores"] = oracle.threads()
    if big:
        out["metrics"] = metrics_leg(run.volume, w.dims)
    del run, cube
    torch.cuda.empty_cache()
    return out


def cpu_baseline_leg(w, gpu_flat, dt, k_ref, planes=(60, 140)):
    """The oracle port on the host cores over a bounded voxel sample (whole
    x-planes of the same volume), plus GPU-vs-oracle parity on that sample."""
    import oracle
    from paper_2506_23568_b200.bpa import region_grid
    cube = _host_cube(gpu_flat.device, w)
    t_rc = time.perf_counter()
    prof = oracle.range_compress(cube, w.upsample)
    t_rc = time.perf_counter() - t_rc
    origin, step = region_grid(w.region, w.dims)
    nx, ny, nz = w.dims
    iy, iz = np.meshgrid(np.arange(ny), np.arange(nz), indexing="ij")
    pts, idx = [], []
    for ix in planes:
        pts.append(np.stack([origin[0] + step[0] * np.full(iy.size, ix),
                             origin[1] + step[1] * iy.ravel(),
                             origin[2] + step[2] * iz.ravel()], axis=-1))
        idx.append((ix * ny + iy.ravel()) * nz + iz.ravel())
    pts = np.concatenate(pts)
    idx = np.concatenate(idx)
    oracle.bp_gather(pts[:64], prof.elements, prof.envelopes, 0.0, prof.dt, prof.k_ref)  # warm
    t = time.perf_counter()
    want, oow = oracle.bp_gather(pts, prof.elements, prof.envelopes, 0.0, prof.dt, prof.k_ref)
    t = time.perf_counter() - t
    units = float(pts.shape[0]) * w.n_elements
    got = gpu_flat.cpu().numpy()[idx]
    rel = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    cb = {"value": round(units / t / 1e9, 4), "unit": UNIT, "cores": oracle.threads(),
          "kind": "port",
          "sample": f"{pts.shape[0]} voxels (x-plane(s) {list(planes)}) x {w.n_elements} elements "
                    f"= {units:.3e} units in {t:.1f} s; range compression of the full cube "
                    f"{t_rc:.1f} s excluded",
          "cpu": _cpu_model()}
    return cb, {"sample_rel_l2_vs_oracle": rel, "sample_voxels": int(pts.shape[0])}


def _host_cube(device, w):
    from paper_2506_23568_b200 import _native
    from paper_2506_23568_b200.model import DataCube
    vals = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                            w.freqs.k_samples, device=device).cpu().numpy()
    return DataCube(values=vals, aperture=w.aperture, freqs=w.freqs)


def _cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args):
    """The reference algorithm's CPU implementation (oracle port of the Numba
    backprojection loop) on all host cores, one bounded voxel sample per step."""
    world, rank, _ = _dist_env()
    if rank != 0:
        return None
    import oracle
    from paper_2506_23568_b200 import workloads
    from paper_2506_23568_b200.bpa import region_grid
    w = make_workload()
    cube = _sim_cpu(w)
    prof = oracle.range_compress(cube, w.upsample)
    origin, step = region_grid(w.region, w.dims)
    nx, ny, nz = w.dims
    iy, iz = np.meshgrid(np.arange(ny), np.arange(nz), indexing="ij")
    rows = max(1, int(args.ref_rows))
    pts = np.stack([origin[0] + step[0] * np.full(rows * nz, nx // 2),
                    origin[1] + step[1] * iy[:rows].ravel(),
                    origin[2] + step[2] * iz[:rows].ravel()], axis=-1)
    units = float(pts.shape[0]) * w.n_elements
    for _ in range(args.warmup):
        oracle.bp_gather(pts[:32], prof.elements, prof.envelopes, 0.0, prof.dt, prof.k_ref)
    t = time.perf_counter()
    for _ in range(args.steps):
        oracle.bp_gather(pts, prof.elements, prof.envelopes, 0.0, prof.dt, prof.k_ref)
    s = (time.perf_counter() - t) / args.steps
    value = units / s / 1e9
    return {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(s * 1e3, 2),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64/c128", "data": "synthetic (seeded Born simulation, numpy)",
            "impl": "reference",
            "config": {"workload": "BASELINE config 1: direct BPA, 32,000 elements, 200x200x64",
                       "sample": f"{pts.shape[0]} voxels x {w.n_elements} elements per step"},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": oracle.threads(),
                             "kind": "port",
                             "sample": f"{pts.shape[0]} voxels x {w.n_elements} elements "
                                       f"= {units:.3e} units per step", "cpu": _cpu_model()},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def _sim_cpu(w):
    """Born cube on the CPU (oracle C loop, OpenMP) for the reference arm."""
    import oracle
    from paper_2506_23568_b200.model import DataCube
    vals = oracle.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                           w.freqs.k_samples)
    return DataCube(values=vals.astype(np.complex64), aperture=w.aperture, freqs=w.freqs)


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-hhffbpa", action="store_true",
                    help="skip the HHFFBPA (configs 2 and 3) extra object")
    ap.add_argument("--ref-rows", type=int, default=64,
                    help="reference arm: y-rows (x 64 z-voxels) of one x-plane per step")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    # no cyclic-GC pauses inside the timed regions (reference counting still
    # frees every per-step buffer); the process is short-lived
    gc.collect()
    gc.disable()
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None:
        print(json.dumps(res))


if __name__ == "__main__":
    main()
