"""Multi-process (world_size 2, gloo, CPU) check of the sharded DFC-Proj host logic:
blocks sharded over ranks, per-rank F step, basis broadcast, per-rank projection, row gather.
Compute is the CPU oracle here (the GPU path plugs the C ABI into the same functions)."""
import os
import socket

import numpy as np
import pytest

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _svd_basis(est):
    # svd_of_product(left, right).U with the reference's numerical-rank cutoff (sketch.hpp:73-86)
    if est.rank == 0:
        return np.zeros((est.left.shape[0], 0))
    ql, rl = np.linalg.qr(est.left)
    qr, rr = np.linalg.qr(est.right)
    u, s, _ = np.linalg.svd(rl @ rr.T)
    keep = int(np.sum(s > 1e-12 * max(est.left.shape[0], est.right.shape[0]) * s[0]))
    return ql @ u[:, :keep]


def _project(Ub, est):
    if est.rank == 0:
        return np.zeros((est.right.shape[0], Ub.shape[1]))
    return est.right @ (Ub.T @ est.left).T


def _worker(rank, world, port, out_path):
    import torch.distributed as dist

    from paper_1107_0789_b200.distributed import column_project_distributed, shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L0, obs = O.gen_mc_instance(120, 90, 3, 5000, 0.1, 3, 0)
    t, seed = 4, 5
    groups = O.partition_columns(seed, 0xDFC0000000000001, 90, t)
    local = {}
    for g in shard(t, world, rank):
        blk = O.extract_columns(obs, groups[g])
        local[g], _ = O.apg_mc(blk)
    res = column_project_distributed(dist, groups, local, 120, _svd_basis, _project)
    if rank == 0:
        ref, _ = O.dfc_run(obs, "proj", t=t, seed=seed)
        got = res[0] @ res[1].T
        err = np.linalg.norm(got - ref.dense()) / np.linalg.norm(ref.dense())
        with open(out_path, "w") as f:
            f.write(repr(float(err)))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_dfc_proj_matches_single_process(tmp_path):
    import torch.multiprocessing as mp

    out = str(tmp_path / "err.txt")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    err = float(open(out).read())
    assert err < 1e-10, err


def _worker_nys(rank, world, port, out_path):
    import torch.distributed as dist

    from paper_1107_0789_b200.distributed import nystrom_distributed, shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, n, l, d, seed = 120, 90, 30, 40, 5
    L0, obs = O.gen_mc_instance(m, n, 3, 5000, 0.1, 3, 0)
    # dfc_nys's D step (P/include/dfc/dfc.hpp:250-290): sorted row / column samples
    rows = np.sort(O.sample_without_replacement(seed, 0xDFC0000000000002, m, d))
    cols = np.sort(O.sample_without_replacement(seed, 0xDFC0000000000003, n, l))
    subs = {0: lambda: O.extract_columns(obs, cols), 1: lambda: O.extract_rows(obs, rows)}
    local = {g: O.apg_mc(subs[g]())[0] for g in shard(2, world, rank)}
    res = nystrom_distributed(dist, local, rows, cols, O.gen_nystrom, O.Estimate)
    if rank == 0:
        ref, _ = O.dfc_run(obs, "nys", l=l, d=d, seed=seed)
        err = np.linalg.norm(res.dense() - ref.dense()) / np.linalg.norm(ref.dense())
        with open(out_path, "w") as f:
            f.write(repr(float(err)))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_dfc_nys_matches_single_process(tmp_path):
    """DFC-Nys with its two subproblems on two ranks (R-hat's factors broadcast to rank 0)."""
    import torch.multiprocessing as mp

    out = str(tmp_path / "err.txt")
    mp.spawn(_worker_nys, args=(2, _free_port(), out), nprocs=2, join=True)
    err = float(open(out).read())
    assert err < 1e-10, err


def test_shard_covers_blocks_once():
    from paper_1107_0789_b200.distributed import shard

    for t in (1, 4, 8, 64):
        for world in (1, 2, 4, 8):
            got = sorted(g for r in range(world) for g in shard(t, world, r))
            assert got == list(range(t))
