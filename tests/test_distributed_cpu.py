"""Multi-rank host logic of libdfcg's distributed path on CPU (no GPU needed):

* the LPT assignment every rank computes (dfcg_assign_blocks) against a plain restatement;
* the host-callback transport (dfcg_comm_init_host) at world size 2 and 3 over gloo: every root
  broadcasts, a ring of point-to-point messages — the traffic the distributed combine sends
  through it (csrc/dist.cpp), driven through the C ABI from torch.distributed callbacks.

The distributed dfc_run itself (same result as the single-process dfc_run) needs device
memory: tests/test_gpu_dist.py runs it with two ranks sharing one GPU over this transport, and
with NCCL at world size 1.
"""
import os
import socket

import numpy as np
import pytest

from paper_1107_0789_b200.distributed import Comm, assign_blocks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def lpt_reference(nnz, nranks):
    order = sorted(range(len(nnz)), key=lambda g: (-nnz[g], g))
    load, count, owner = [0] * nranks, [0] * nranks, [0] * len(nnz)
    for g in order:
        best = min(range(nranks), key=lambda q: (load[q], count[q], q))
        owner[g] = best
        load[best] += max(nnz[g], 0)
        count[best] += 1
    return owner


def test_lpt_assignment_matches_restatement():
    rng = np.random.default_rng(5)
    cases = [[5, 5, 5, 5], [0, 0, 7], [1250000] * 8, list(rng.zipf(1.5, 64)), list(rng.integers(0, 10**7, 13))]
    for nnz in cases:
        for nranks in (1, 2, 3, 4, 8):
            got = assign_blocks(nnz, nranks)
            assert got == lpt_reference(list(map(int, nnz)), nranks), (nnz, nranks)
            assert all(0 <= o < nranks for o in got)
    # balanced c2 shape: 8 equal blocks over 8, 4, 2 ranks -> equal counts per rank
    for nranks in (2, 4, 8):
        got = assign_blocks([1250000] * 8, nranks)
        assert sorted(np.bincount(got, minlength=nranks)) == [8 // nranks] * nranks
    # Zipf-skewed blocks: LPT's makespan within 4/3 of the lower bound
    nnz = [int(x) for x in np.random.default_rng(9).zipf(1.3, 64) * 1000]
    for nranks in (2, 4, 8):
        got = assign_blocks(nnz, nranks)
        loads = np.bincount(got, weights=nnz, minlength=nranks)
        assert loads.max() <= 4 / 3 * max(sum(nnz) / nranks, max(nnz)) + 1
    with pytest.raises(ValueError):
        assign_blocks([1, 2], 0)


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = Comm.host()
    bad = comm.selftest()
    comm.close()
    with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as f:
        f.write(str(bad))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_transport_through_c_abi(tmp_path, world):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert open(tmp_path / f"r{r}.txt").read() == "0", r
