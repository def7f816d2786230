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


def _comm_worker(rank, world, port, out_path):
    sys.path.insert(0, str(REPO))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_23568_b200.dist import TorchComm, plan_shard
    comm = TorchComm()
    # uneven complex segments: rank r owns [starts[r], starts[r+1])
    starts = [0, 5, 17, 18, 30][:world + 1]
    buf = torch.zeros(starts[-1], dtype=torch.complex64)
    a, b = starts[rank], starts[rank + 1]
    buf[a:b] = torch.arange(a, b, dtype=torch.float32) * (1 + 1j)
    segs = list(zip(starts[:-1], starts[1:]))
    # gather to root: rank 0 passes the whole buffer, the others only their
    # own segment (indexed from its start)
    own = buf[a:b].clone()
    root_buf = buf.clone() if rank == 0 else own
    comm.gather_segments(root_buf, segs, base=0 if rank == 0 else a)
    comm.allgather_segments(buf, segs)
    cnt = torch.tensor([rank + 1, 10 * rank], dtype=torch.int64)
    comm.allreduce_sum(cnt)
    # split_top's sums: uint8 masks and float64 positions, each point owned by
    # one rank (the others hold zeros), on views into larger pools
    pool_v = torch.zeros(12, dtype=torch.uint8)
    pool_p = torch.zeros((12, 3), dtype=torch.float64)
    mine = torch.arange(12) % world == rank
    pool_v[4:][mine[4:]] = 1
    pool_p[4:][mine[4:]] = torch.arange(8, dtype=torch.float64)[mine[4:]].unsqueeze(1) + 0.25
    comm.allreduce_sum(pool_v[4:])
    comm.allreduce_sum(pool_p[4:])
    # the subtree plan every rank derives must tile the leaves / elements
    plans = [plan_shard(1000, 8, 2, world, r) for r in range(world)]
    if rank == 0:
        np.save(out_path, {"buf": buf.numpy(), "root": root_buf.numpy(), "cnt": cnt.numpy(),
                           "pool_v": pool_v.numpy(), "pool_p": pool_p.numpy(),
                           "rows": [p[3] for p in plans], "kx": [p[1] for p in plans]},
                allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_comm_segments_allreduce_and_plan(tmp_path, world):
    out = tmp_path / "r.npy"
    mp.start_processes(_comm_worker, args=(world, _free_port(), str(out)), nprocs=world,
                       start_method="spawn", join=True)
    res = np.load(out, allow_pickle=True).item()
    n = [0, 5, 17, 18, 30][world]
    assert np.array_equal(res["buf"], np.arange(n) * (1 + 1j))
    assert np.array_equal(res["root"], np.arange(n) * (1 + 1j))
    assert list(res["cnt"]) == [sum(range(1, world + 1)), 10 * sum(range(world))]
    assert list(res["pool_v"]) == [0] * 4 + [1] * 8
    assert np.array_equal(res["pool_p"][4:], np.repeat(np.arange(8.0)[:, None] + 0.25, 3, 1))
    assert not res["pool_p"][:4].any()
    rows = res["rows"]
    assert rows[0][0] == 0 and rows[-1][1] == 1000
    assert all(rows[r][1] == rows[r + 1][0] for r in range(world - 1))
    assert len(set(res["kx"])) == 1 and res["kx"][0] >= 0


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
