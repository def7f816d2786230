"""Multi-process (world_size 2, gloo, CPU) test of the voxel-sharding logic
used for N>1 GPUs: each rank computes its contiguous voxel slab and the
all-gather reassembles the volume exactly.  The per-rank compute here is the
CPU oracle (test infrastructure), standing in for the CUDA kernel that the
GPU path plugs into the same ``run_voxel_sharded``."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_path):
    sys.path.insert(0, str(REPO))
    sys.path.insert(0, str(REPO / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), ORACLE_THREADS="2")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from goldens import load
    from paper_2506_23568_b200.bpa import region_grid
    from paper_2506_23568_b200.dist import run_voxel_sharded
    case = load("small")
    dims = case.dims
    origin, step = region_grid(case.region, dims)
    prof = oracle.range_compress(case.cube, 8)
    axes = [origin[a] + step[a] * np.arange(dims[a]) for a in range(3)]
    pts = np.stack([m.ravel() for m in np.meshgrid(*axes, indexing="ij")], axis=-1)

    def compute(vb, ve):
        vals, _ = oracle.bp_gather(pts[vb:ve], prof.elements, prof.envelopes, prof.t0, prof.dt,
                                   prof.k_ref)
        return torch.from_numpy(vals.astype(np.complex64))

    full = run_voxel_sharded(int(np.prod(dims)), compute)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_voxel_sharded_gather_reassembles_volume(tmp_path, world):
    out = tmp_path / "vol.npy"
    mp.start_processes(_worker, args=(world, _free_port(), str(out)), nprocs=world,
                       start_method="spawn", join=True)
    got = np.load(out)
    sys.path.insert(0, str(REPO / "tests"))
    from goldens import load, rel_l2
    case = load("small")
    want = case.z["bpa"].ravel()
    assert got.shape == want.shape
    assert rel_l2(got, want) < 1e-6
