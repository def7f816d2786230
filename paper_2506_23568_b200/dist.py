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

import numpy as np

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


def _allreduce_sum(t, group=None):
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        t = t.clone()
        dist.all_reduce(t, group=group)
    return t
