"""Multi-GPU plumbing: one process per GPU, torch.distributed over NCCL.

BPA (BASELINE config 1) and the final HHFFBPA landing are pointwise in the
output voxels, so the volume is sharded by contiguous ranges of the
flattened [nx][ny][nz] index (x-slabs of whole y-z planes, balanced to within
one voxel); every rank holds all echo profiles (each rank range-compresses
its own copy of the cube -- cheaper than a broadcast of the 4-8x larger
profiles).  The only data-path collective is the final gather of the voxel
slabs: one ``all_gather_into_tensor`` of equal-size complex64 chunks (NCCL
over NVLink/NVSwitch).  ``run_voxel_sharded`` is backend-agnostic so the
sharding and reassembly logic is tested with gloo on CPU
(tests/test_dist_gloo.py).
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np

from .errors import ConfigError
from .bpa import (_finish, bpa_volume_device, check_delay_window, default_grid_dims,
                  el_f32x4, region_grid)
from .model import validate_geometry
from .rangecomp import range_compress


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous [begin, end) of n items for ``rank``."""
    base, extra = divmod(int(n), int(world))
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def chunk_size(n: int, world: int) -> int:
    return -(-int(n) // int(world))


def run_voxel_sharded(n_vox: int, compute, group=None, device=None, dtype=None):
    """Compute this rank's voxel range with ``compute(vb, ve) -> 1-D tensor``
    and all-gather the slabs; returns the full flat volume on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    vb, ve = shard_range(n_vox, rank, world)
    part = compute(vb, ve)
    if world == 1:
        return part
    c = chunk_size(n_vox, world)
    send = torch.zeros(c, dtype=part.dtype, device=part.device)
    send[:ve - vb] = part
    recv = torch.empty(c * world, dtype=part.dtype, device=part.device)
    if part.is_complex() and not dist.get_backend(group) == "nccl":
        # gloo has no complex all_gather; move the raw float pairs instead
        rv = torch.view_as_real(recv)
        dist.all_gather_into_tensor(rv, torch.view_as_real(send), group=group)
    else:
        dist.all_gather_into_tensor(recv, send, group=group)
    pieces = [recv[r * c: r * c + (shard_range(n_vox, r, world)[1] - shard_range(n_vox, r, world)[0])]
              for r in range(world)]
    return torch.cat(pieces)


def bpa_reconstruct_sharded(cube, region, dims=None, upsample: int = 8, group=None):
    """bpa_reconstruct over all ranks of ``group``: every rank returns the
    same ImageVolume (the gathered volume)."""
    validate_geometry(cube.aperture, region)
    if dims is None:
        dims = default_grid_dims(region, cube.freqs)
    dims = tuple(int(d) for d in dims)
    origin, step = region_grid(region, dims)
    prof = range_compress(cube, upsample)
    check_delay_window(prof, region)
    el4 = el_f32x4(prof.elements_dev)
    oows = []

    def compute(vb, ve):
        vol, oow = bpa_volume_device(prof.envelopes, el4, region, dims, prof.t0, prof.dt,
                                     prof.k_ref, vox_range=(vb, ve))
        oows.append(oow)
        return vol

    flat = run_voxel_sharded(int(np.prod(dims)), compute, group)
    oow = _allreduce_sum(oows[0], group)
    return _finish(flat, oow, dims, origin, step,
                   {"algorithm": "bpa", "upsample": upsample, "dims": list(dims)})[0]


# ---------------------------------------------------------------------------
# HHFFBPA across GPUs
# ---------------------------------------------------------------------------

class TorchComm:
    """Collectives over torch.distributed: NCCL on GPUs; with a host backend
    (gloo) device tensors are staged through host memory -- the CPU tests'
    and a debug mode's path (several ranks sharing one GPU, where no kernel
    may wait on another rank)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.host_stage = dist.is_initialized() and dist.get_backend(group) != "nccl"

    def _raw(self, t):
        import torch
        return torch.view_as_real(t) if t.is_complex() else t

    def _host(self, t):
        return t.cpu() if self.host_stage and t.is_cuda else t

    def allreduce_sum(self, t) -> None:
        import torch.distributed as dist
        if self.world > 1:
            h = self._host(t)
            dist.all_reduce(h, group=self.group)
            if h is not t:
                t.copy_(h)

    def allgather_segments(self, buf, segments) -> None:
        """buf[a_r:b_r] holds rank r's data on rank r; afterwards every rank
        holds every segment (one all_gather of equal padded chunks)."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return
        longest = max(b - a for a, b in segments)
        a, b = segments[self.rank]
        send = torch.zeros(longest, dtype=buf.dtype, device=buf.device)
        send[:b - a] = buf[a:b]
        send = self._host(send)
        recv = torch.empty(longest * self.world, dtype=buf.dtype, device=send.device)
        dist.all_gather_into_tensor(self._raw(recv), self._raw(send), group=self.group)
        for r, (a, b) in enumerate(segments):
            if r != self.rank:
                buf[a:b] = recv[r * longest: r * longest + (b - a)].to(buf.device)

    def gather_segments(self, buf, segments, root: int = 0, base: int = 0) -> None:
        """Like allgather_segments, but only ``root`` receives the other
        ranks' segments (NCCL gather: root takes in (W-1)/W of the buffer,
        the other ranks only send).  ``buf`` holds global indices from
        ``base`` on (a non-root rank may pass just its own segment)."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return
        longest = max(b - a for a, b in segments)
        a, b = segments[self.rank]
        send = torch.zeros(longest, dtype=buf.dtype, device=buf.device)
        send[:b - a] = buf[a - base:b - base]
        send = self._host(send)
        if self.rank == root:
            parts = [torch.empty(longest, dtype=buf.dtype, device=send.device)
                     for _ in range(self.world)]
            dist.gather(self._raw(send), [self._raw(p) for p in parts], dst=root,
                        group=self.group)
            for r, (a, b) in enumerate(segments):
                if r != self.rank:
                    buf[a - base:b - base] = parts[r][:b - a].to(buf.device)
        else:
            dist.gather(self._raw(send), None, dst=root, group=self.group)


class EmulatedComm:
    """World of `world` ranks emulated by host threads in one process on one
    GPU (for tests): each rank runs its own pipeline; collectives exchange
    tensors through host-side barriers -- no kernel ever waits on another."""

    def __init__(self, rank: int, world: int, shared: dict):
        import threading
        self.rank, self.world = rank, world
        self.shared = shared
        shared.setdefault("barrier", threading.Barrier(world))
        shared.setdefault("slots", [None] * world)

    def _exchange(self, t):
        import torch
        torch.cuda.synchronize()
        self.shared["slots"][self.rank] = t
        self.shared["barrier"].wait()
        out = list(self.shared["slots"])
        self.shared["barrier"].wait()
        return out

    def allreduce_sum(self, t) -> None:
        parts = self._exchange(t.clone())
        total = parts[0].clone()
        for p in parts[1:]:
            total += p
        t.copy_(total)

    def gather_segments(self, buf, segments, root: int = 0, base: int = 0) -> None:
        a, b = segments[self.rank]
        parts = self._exchange(buf[a - base:b - base].clone())
        if self.rank == root:
            for r, (a, b) in enumerate(segments):
                if r != self.rank:
                    buf[a - base:b - base] = parts[r]

    def allgather_segments(self, buf, segments) -> None:
        a, b = segments[self.rank]
        parts = self._exchange(buf[a:b].clone())
        for r, (a, b) in enumerate(segments):
            if r != self.rank:
                buf[a:b] = parts[r]


def exchange_level(sched, world: int):
    """Highest grid level (index into sched.level_slices) whose subimage
    count is a multiple of `world`: each rank owns count/world consecutive
    subtrees below it.  None when no level splits evenly."""
    best = None
    for k, (a, b) in enumerate(sched.level_slices):
        if (b - a) % world == 0 and b - a >= world:
            best = k
    return best


def plan_shard(n_elements: int, levels: int, merge_factor: int, world: int, rank: int):
    """(schedule, exchange level kx, owned grid slices per level <= kx,
    owned element rows [e0, e1)).  kx = -1 when no level splits evenly (then
    every rank builds every subtree and only the landing is sharded)."""
    from .ffbp import Schedule
    sched = Schedule.shared(int(n_elements), levels, merge_factor)
    n_lv = len(sched.level_slices)
    kx = exchange_level(sched, world) if world > 1 else n_lv - 1
    if kx is None:
        return sched, -1, list(sched.level_slices), (0, n_elements)
    owned = []
    for k in range(kx + 1):
        a, b = sched.level_slices[k]
        per = (b - a) // world
        owned.append((a + rank * per, a + (rank + 1) * per))
    g0, g1 = owned[0]
    e0 = int(sched.grids["start"][g0])
    e1 = int(sched.grids["stop"][g1 - 1])
    return sched, kx, owned, (e0, e1)


OUTPUTS = ("all", "root", "shard")


def owned_elements(n_elements: int, levels: int, merge_factor: int = 2, comm=None):
    """Element rows [e0, e1) whose echoes this rank needs (its subaperture
    group): a multi-process caller loads only these rows and
    passes them as ``rows=`` to hhffbpa_reconstruct_sharded."""
    comm = comm or TorchComm()
    return plan_shard(n_elements, levels, merge_factor, comm.world, comm.rank)[3]


def hhffbpa_reconstruct_sharded(cube, region, final_dims=None, params=None, upsample: int = 8,
                                merge_factor: int = 2, comm=None, output: str = "all",
                                rows=None, split_top: bool = False):
    """hhffbpa_reconstruct (ffbp.py:415-513) over all ranks of `comm`
    (default: torch.distributed's world).  Each rank transfers and
    range-compresses only its own subaperture group's echoes (streamed in
    chunks, the compression overlapping the upload).

    ``output`` -- where the volume lands:
      "all"   every rank returns the whole ImageVolume (NCCL all-gather);
      "root"  rank 0 returns the whole volume (NCCL gather), the others their
              own x-slab;
      "shard" every rank returns its own x-slab only (no volume collective;
              the slabs tile the volume, see ``ShardedVolume``).
    Provenance and error checks are identical on every rank in all modes.

    ``rows``: this rank's echo rows [e0, e1) only (owned_elements()), e.g.
    a pinned host buffer each process filled itself; ``cube.values`` is then
    never read (each process holds 1/W of the cube).
    ``split_top``: see hhffbpa_sharded_device (the top grids' Newton split by
    u-rows across ranks instead of run whole on every rank).
    """
    import torch
    from .bpa import _finish, check_delay_window, default_grid_dims, region_grid
    from .ffbp import FfbpParams, check_grids, default_levels, provenance_of
    from .model import leaf_bounds, validate_geometry
    from .rangecomp import CubeUpload, RangeProfileSet, profile_axis
    if output not in OUTPUTS:
        raise ConfigError(f"output must be one of {OUTPUTS}")
    comm = comm or TorchComm()
    params = params or FfbpParams()
    validate_geometry(cube.aperture, region)
    kgrid = cube.freqs
    dims = tuple(int(d) for d in (final_dims or default_grid_dims(region, kgrid)))
    levels = params.levels if params.levels is not None else default_levels(cube.aperture)
    if levels < 2:
        raise ConfigError("the sharded HHFFBPA needs levels >= 2 (levels=1 is the BPA: "
                          "use bpa_reconstruct_sharded)")
    if region.z_min <= 0.0:
        raise ConfigError("region must sit strictly in front of the array")
    leaf_bounds(cube.aperture.n_elements, levels)  # ConfigError when too deep
    n_el = cube.aperture.n_elements
    _, _, _, (e0, e1) = plan_shard(n_el, levels, merge_factor, comm.world, comm.rank)
    el_dev = torch.tensor(np.ascontiguousarray(cube.aperture.elements, dtype=np.float64),
                          device="cuda")
    n_t, dt, k_ref, _ = profile_axis(kgrid, upsample)
    window = RangeProfileSet(envelopes=torch.empty((0, n_t)), t0=0.0, dt=dt,
                             upsample=upsample, k_ref=k_ref, aperture=cube.aperture,
                             freqs=kgrid, elements_dev=el_dev)
    check_delay_window(window, region)
    if rows is not None and tuple(rows.shape) != (e1 - e0, kgrid.count):
        raise ConfigError(f"rows must hold this rank's elements [{e0}, {e1}) x "
                          f"{kgrid.count} frequencies, got {tuple(rows.shape)}")
    uploads = []

    def start_upload():
        # started once the plan's small copy is queued (it must not wait behind
        # the cube's chunks in the copy engine)
        if rows is not None:
            up = CubeUpload(rows)
            up.row0 = e0
            up.chunks = [(a + e0, b + e0, ev) for a, b, ev in up.chunks]
        else:
            up = CubeUpload(cube.values, rows=(e0, e1))
        uploads.append(up)
        return up

    res = hhffbpa_sharded_device(comm, None, e0, el_dev, kgrid, region, dims, params,
                                 levels, merge_factor, upsample, output=output,
                                 upload=start_upload, split_top=split_top)
    if int(res.oow.cpu()[0]):  # a leaf delay outside the range gate (all-reduced: every rank agrees)
        res = hhffbpa_sharded_device(comm, uploads[0].tensor, e0, el_dev, kgrid, region, dims,
                                     params, levels, merge_factor, upsample, gate=False,
                                     output=output, split_top=split_top)
    origin, step = region_grid(region, dims)
    extra = torch.cat([res.flags, res.stats.reshape(-1)])
    whole = output == "all" or (output == "root" and comm.rank == 0)
    vol_dims = dims if whole else (res.vox_range[1] - res.vox_range[0], 1, 1)
    volume, tail = _finish(res.volume, res.oow, vol_dims, origin, step, {}, extra)
    fl = tail[:res.flags.numel()]
    st = tail[res.flags.numel():].reshape(-1, res.stats.shape[1])
    run = SimpleNamespace(sched=res.sched, lattices=SimpleNamespace(descs=res.descs))
    check_grids(run, st)
    prov = provenance_of(run, st, fl, dims, params, levels, upsample, merge_factor)
    if not whole:
        return ShardedVolume(values=volume.values.reshape(-1), vox_range=res.vox_range, dims=dims,
                             origin=origin, step=step, provenance=prov)
    object.__setattr__(volume, "provenance", prov)
    return volume


class ShardedVolume(SimpleNamespace):
    """One rank's x-slab of a voxel-sharded volume: ``values`` complex64 for
    the flattened [nx][ny][nz] indices ``vox_range`` = [vb, ve) of the whole
    grid ``dims`` (origin / step as ImageVolume's); ``provenance`` is the
    whole reconstruction's."""

    def flat_indices(self):
        return np.arange(*self.vox_range)


def hhffbpa_sharded_device(comm, cube_dev_rows, e_row0: int, el_dev, kgrid, region, final_dims,
                           params, levels: int, merge_factor: int, upsample: int,
                           gate: bool = True, output: str = "all", upload=None,
                           plan_cache=None, split_top: bool = False):
    """One rank's share of HHFFBPA:

    1. subaperture-group partition: the rank owns a contiguous run of
       subtrees up to the exchange level and range-compresses only those
       elements (``cube_dev_rows`` = its rows, starting at ``e_row0``), only
       the delay bins the leaf stage can read (the plan's range gate, as in
       ffbp.hhffbpa_from_cube; ``gate=False``: full profiles);
       every grid is PLANNED for the whole region on every rank (so lattices
       are identical to the 1-GPU ones), Newton runs only where this rank
       evaluates points;
    2. all-gather of the exchange level's downconverted lattices (NCCL);
    3. the few top merge levels redundantly on every rank;
    4. the Cartesian landing voxel-sharded, then (``output``) an all-gather
       of the slabs ("all"), a gather to rank 0 ("root") or nothing
       ("shard").

    ``split_top``: the grids above the exchange level (planned and merged
    by every rank) are inverted split by lattice u-rows across the ranks
    (grid build) and their positions / masks / counters summed
    with one all-reduce, instead of every rank inverting them whole.

    ``upload`` (rangecomp.CubeUpload of this rank's rows, or a zero-argument
    factory of one started right after the plan is queued; ``cube_dev_rows``
    may then be None): compress chunk by chunk as rows land.  ``plan_cache``
    (the ``plan`` of an earlier call of this rank with the same geometry):
    no host wait on the plan (ffbp.PlanCache).  Returns a namespace: volume
    (flat complex64: the whole volume where it was gathered, else this
    rank's slab), vox_range, stats[G,6], flags, oow (identical on all
    ranks), sched, descs, plan (this rank's PlanCache).
    """
    import torch
    from .bpa import el_f32x4
    from .ffbp import (Pipeline, PlanCache, finish_lattices,
                       geometry_stream, plan_lattices, src_pad_of)
    from .rangecomp import profile_axis, range_compress_device, range_compress_window
    world, rank = comm.world, comm.rank
    sched, kx, owned, _ = plan_shard(el_dev.shape[0], levels, merge_factor, world, rank)
    n_lv = len(sched.level_slices)
    mask = np.zeros(sched.n_grids, dtype=bool)
    for k in range(n_lv):
        a, b = owned[k] if k <= kx else sched.level_slices[k]
        mask[a:b] = True
    n_t, dt, _, _ = profile_axis(kgrid, upsample)
    window_hi = (n_t - 1) * dt
    g_top = sched.level_slices[kx][1] if kx >= 0 else sched.n_grids  # first grid above
    split_top = bool(split_top) and world > 1 and kx >= 0 and g_top < sched.n_grids
    row_split = (rank, world, range(g_top, sched.n_grids)) if split_top else None
    # as ffbp.hhffbpa_from_cube: plan and Newton on the high-priority
    # geometry stream, the (gated) range compression on the caller's stream
    # beside Newton
    main = torch.cuda.current_stream()
    geo = geometry_stream(el_dev.device)
    geo.wait_stream(main)
    with torch.cuda.stream(geo):
        pending = plan_lattices(el_dev, sched, region, kgrid, params.gamma, params.margin,
                                src_pad_of(params), window_hi, gate_dt=dt if gate else None,
                                gate_bins=n_t, cached=plan_cache)
    if callable(upload):
        upload = upload()
        cube_dev_rows = upload.tensor
    lat = None
    if gate:
        if plan_cache is None:
            pending["done"].synchronize()
        n_cols, b0, w = (int(v) for v in pending["host_s"][16:40].view(np.int64))
        with torch.cuda.stream(geo):  # Newton first, as the 1-GPU step (ffbp)
            lat = finish_lattices(pending, newton_grids=mask, row_split=row_split)
        env, t0, dt, k_ref = range_compress_window(
            cube_dev_rows, kgrid, upsample, b0, w, chunks=upload.chunks if upload else None,
            row0=e_row0)
    else:
        if upload is not None:
            upload.wait()
        env, dt, k_ref = range_compress_device(cube_dev_rows, kgrid, upsample)
        t0 = 0.0
    if lat is None:
        with torch.cuda.stream(geo):
            lat = finish_lattices(pending, newton_grids=mask, row_split=row_split)
    main.wait_stream(geo)
    if split_top:
        # each top-grid point was inverted by exactly one rank: sum the
        # shares (the positions pool is uninitialised where a rank did not
        # invert, so every rank zeroes the rows it left to the others first
        # -- on the geometry stream, ahead of nothing: Newton has run)
        p0 = int(lat.descs["offset"][g_top])
        p1 = int(lat.descs["offset"][-1] + lat.npts[-1])
        top_pos = lat.positions[p0:p1]
        own = lat.valid[p0:p1] != 0
        top_pos.mul_(own.unsqueeze(1).to(top_pos.dtype))
        comm.allreduce_sum(top_pos)
        comm.allreduce_sum(lat.valid[p0:p1])
        top_stats = lat.stats[g_top:]
        comm.allreduce_sum(top_stats)
    for t in (lat.positions, lat.valid, lat.stats, lat.keep[1]):
        t.record_stream(main)
    pipe = Pipeline(env, el_dev, el_f32x4(el_dev), t0, dt, k_ref, kgrid, region, final_dims,
                    params, levels, merge_factor, window_hi, newton_grids=mask,
                    env_row0=e_row0, sched=sched, lat=lat)
    pipe.leaves(*owned[0])
    for k in range(max(kx, 0)):
        pipe.merge(k, *owned[k + 1])
    if kx >= 0 and world > 1:
        a, b = sched.level_slices[kx]
        per = (b - a) // world
        off = pipe.lat.descs["offset"].astype(np.int64)
        npts = pipe.lat.npts
        segs = [(int(off[a + r * per]), int(off[a + (r + 1) * per - 1] + npts[a + (r + 1) * per - 1]))
                for r in range(world)]
        comm.allgather_segments(pipe.values, segs)
    for k in range(max(kx, 0), pipe.n_stages):
        pipe.merge(k)
    n_vox = int(np.prod(final_dims))
    vb, ve = shard_range(n_vox, rank, world)
    part = pipe.land((vb, ve))
    # volume slabs
    segs = [shard_range(n_vox, r, world) for r in range(world)]
    if output == "all" or world == 1:
        vol = torch.zeros(n_vox, dtype=torch.complex64, device=part.device)
        vol[vb:ve] = part
        comm.allgather_segments(vol, segs)
    elif output == "root":
        if rank == 0:
            vol = torch.zeros(n_vox, dtype=torch.complex64, device=part.device)
            vol[vb:ve] = part
        else:
            vol = part
        comm.gather_segments(vol, segs, base=0 if rank == 0 else vb)
    else:
        vol = part
    # counters: rows / stages computed by owners are summed, redundant ones kept
    stats = pipe.lat.stats
    if world > 1 and kx >= 0:
        low = stats.clone()
        g_hi = sched.level_slices[kx][1]
        low[g_hi:] = 0
        comm.allreduce_sum(low)
        stats = torch.cat([low[:g_hi], stats[g_hi:]])
        fl = pipe.flags.clone()
        fl[kx:pipe.n_stages] = 0
        comm.allreduce_sum(fl)
        flags = torch.cat([fl[:kx], pipe.flags[kx:pipe.n_stages], fl[pipe.n_stages:]])
        oow = pipe.oow.clone()
        comm.allreduce_sum(oow)
    else:
        flags = pipe.flags.clone()
        fl = flags[pipe.n_stages:].clone()
        comm.allreduce_sum(fl)
        flags[pipe.n_stages:] = fl
        oow = pipe.oow
    whole = output == "all" or world == 1 or (output == "root" and rank == 0)
    plan = plan_cache if plan_cache is not None else PlanCache.of_lattices(pipe.lat)
    return SimpleNamespace(volume=vol, vox_range=(0, n_vox) if whole else (vb, ve), stats=stats,
                           flags=flags, oow=oow, sched=sched, descs=pipe.lat.descs, plan=plan)



def _allreduce_sum(t, group=None):
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        t = t.clone()
        dist.all_reduce(t, group=group)
    return t
