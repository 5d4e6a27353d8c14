"""GPU tests of libdfcg's native multi-GPU dfc_run (dfcg_dfc_run_dist, csrc/dfc_dist.cpp).

* NCCL at world size 1 (the box has one GPU): communicator creation from an ncclUniqueId, the
  distributed combine's code path, result equal to the single-process dfc_run.
* Two ranks sharing one GPU over the host-callback transport (gloo; collectives on the CPU, so
  no rank's kernels wait on another's): each rank solves its LPT share of the subproblems and
  joins the exchange; both ranks return the single-process dfc_run's estimate
  (P/tests/test_dfc.cpp:322-342's scheduling invariance, extended to ranks), for DFC-Proj,
  Proj-Ens (all anchors and 4 anchors), DFC-Nys, Nys-Ens and DFC-RP; a failing subproblem
  raises BlockError with the lowest index on every rank.
"""
import os
import socket

import numpy as np
import pytest

import paper_1107_0789_b200 as P
from paper_1107_0789_b200.distributed import Comm, dfc_run_dist

pytestmark = pytest.mark.gpu

CASES = [
    ("proj", dict(t=5)),
    ("proj", dict(t=5, ensemble=True)),
    ("proj", dict(t=6, ensemble=True, ensemble_anchors=4)),
    ("nys", dict(l=50, d=60)),
    ("nys", dict(l=60, d=50, ensemble=True)),
    ("rp", dict(t=4)),
    ("rp", dict(t=3, ensemble=True)),
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _instance():
    return P.gen_mc_instance(180, 150, 3, 9000, 0.1, 2)


def _rel(a, b):
    A, B = a.dense(), b.dense()
    return float(np.linalg.norm(A - B) / max(np.linalg.norm(B), 1e-300))


def test_nccl_world1_equals_dfc_run():
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = Comm.nccl(device=0)
        L0, obs = _instance()
        for variant, kw in CASES:
            ref, rinfo = P.dfc_run(obs, variant, seed=3, workers=2, **kw)
            est, info = dfc_run_dist(obs, comm, variant, seed=3, workers=2, **kw)
            assert est.rank == ref.rank, (variant, kw)
            assert _rel(est, ref) <= 1e-12, (variant, kw, _rel(est, ref))
            assert [s.iterations for s in info["subproblems"]] == [s.iterations for s in rinfo["subproblems"]]
            assert set(info["owner"]) == {0}
        comm.close()
    finally:
        dist.destroy_process_group()


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = Comm.host()
    L0, obs = _instance()
    lines = []
    for variant, kw in CASES:
        est, info = dfc_run_dist(obs, comm, variant, seed=3, workers=2, **kw)
        np.savez(os.path.join(out_dir, f"{variant}_{len(lines)}_r{rank}.npz"), left=est.left, right=est.right,
                 its=np.array([s.iterations for s in info["subproblems"]]), owner=np.array(info["owner"]))
        lines.append(variant)
    # failure propagation: every block fails (invalid solver config) -> BlockError(0) on every rank
    try:
        dfc_run_dist(obs, comm, "proj", t=4, seed=3, solver_cfg=P.ApgConfig(rel_tol=2.0))
        msg = "no error"
    except P.BlockError as e:
        msg = f"{e.block}|{e}"
    with open(os.path.join(out_dir, f"err_r{rank}.txt"), "w") as f:
        f.write(msg)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_on_one_gpu_equal_dfc_run(tmp_path):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    L0, obs = _instance()
    for i, (variant, kw) in enumerate(CASES):
        ref, rinfo = P.dfc_run(obs, variant, seed=3, workers=2, **kw)
        owners = None
        for r in range(2):
            z = np.load(tmp_path / f"{variant}_{i}_r{r}.npz")
            est = P.Estimate(z["left"], z["right"])
            assert _rel(est, ref) <= 1e-12, (variant, kw, r, _rel(est, ref))
            assert list(z["its"]) == [s.iterations for s in rinfo["subproblems"]]
            owners = z["owner"] if owners is None else owners
            assert np.array_equal(owners, z["owner"])
        assert set(owners.tolist()) == {0, 1}, (variant, owners)  # both ranks solved something
    for r in range(2):
        blk, msg = open(tmp_path / f"err_r{r}.txt").read().split("|", 1)
        assert blk == "0" and msg.startswith("block 0: ") and "block 0: block" not in msg, msg
