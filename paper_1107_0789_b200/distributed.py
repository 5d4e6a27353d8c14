"""Multi-GPU DFC-Proj: blocks sharded over ranks, no data-path collective during the solve
(the F-step subproblems are independent, P/include/dfc/dfc.hpp:133-147), and the combine
(column_project, P/include/dfc/sketch.hpp:170-199) split into
    1. the rank owning block 0 computes the basis U_b = svd_of_product(C_1).U and
       broadcasts it (NCCL over NVLink when the process group is "nccl"),
    2. every rank projects its own blocks: R_g = right_g (U_b^T left_g)^T,
    3. the projected rows are gathered to rank 0 and scattered to their original columns.
DFC-Nys (nystrom_distributed): the two subproblems (C-hat, R-hat) solve concurrently on two
ranks; R-hat's factors are broadcast from its rank (the only exchange) and rank 0 combines.
The compute steps are injected (GPU C ABI in bench.py, the CPU oracle in the gloo tests), so
the same host logic runs under both backends.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Sequence

import numpy as np


def shard(t: int, world: int, rank: int) -> List[int]:
    """Blocks owned by `rank`: round-robin over the t plan groups (balanced for t % world == 0)."""
    return [g for g in range(t) if g % world == rank]


def _tensor(dist, a: np.ndarray, device):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def broadcast_array(dist, a: np.ndarray | None, src: int, device, shape_hint=None) -> np.ndarray:
    """Broadcast a float64 2-D array from `src` (shape sent first)."""
    import torch

    rank = dist.get_rank()
    shp = torch.zeros(2, dtype=torch.int64, device=device)
    if rank == src:
        shp[0], shp[1] = a.shape
    dist.broadcast(shp, src)
    r, c = int(shp[0]), int(shp[1])
    buf = _tensor(dist, a, device) if rank == src else torch.empty((r, c), dtype=torch.float64, device=device)
    dist.broadcast(buf, src)
    return buf.cpu().numpy()


def gather_rows(dist, local: Dict[int, np.ndarray], t: int, kb: int, device) -> Dict[int, np.ndarray] | None:
    """Gather per-block row slabs (w_g x kb) to rank 0; all ranks pad to the largest slab."""
    import torch

    world, rank = dist.get_world_size(), dist.get_rank()
    wmax = torch.tensor([max([a.shape[0] for a in local.values()] + [0])], dtype=torch.int64, device=device)
    dist.all_reduce(wmax, op=dist.ReduceOp.MAX)
    w = int(wmax.item())
    slots = (t + world - 1) // world
    mine = np.zeros((slots, w, kb), np.float64)
    for i, g in enumerate(shard(t, world, rank)):
        a = local[g]
        mine[i, : a.shape[0]] = a
    send = _tensor(dist, mine, device)
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send)
    if rank != 0:
        return None
    out = {}
    for r in range(world):
        arr = recv[r].cpu().numpy()
        for i, g in enumerate(shard(t, world, r)):
            out[g] = arr[i]
    return out


def column_project_distributed(dist, groups: Sequence[np.ndarray], local_ests: Dict[int, object], m: int,
                               basis_fn: Callable, project_fn: Callable, device="cpu"):
    """DFC-Proj combine over ranks. local_ests: {g: Estimate} for this rank's blocks.
    basis_fn(est) -> U_b (m x kb); project_fn(U_b, est) -> R_g (w_g x kb).
    Returns (U_b, right) on rank 0, None elsewhere."""
    rank = dist.get_rank()
    t = len(groups)
    n = int(sum(len(g) for g in groups))
    Ub = basis_fn(local_ests[0]) if rank == 0 else None
    Ub = broadcast_array(dist, Ub, 0, device)
    kb = Ub.shape[1]
    if kb == 0:
        return (np.zeros((m, 0)), np.zeros((n, 0))) if rank == 0 else None
    local_rows = {g: project_fn(Ub, e) for g, e in local_ests.items()}
    rows = gather_rows(dist, local_rows, t, kb, device)
    if rank != 0:
        return None
    right = np.zeros((n, kb))
    for g, idx in enumerate(groups):
        right[np.asarray(idx)] = rows[g][: len(idx)]
    return Ub, right


def nystrom_distributed(dist, local_ests: Dict[int, object], rows, cols, nystrom_fn: Callable, make_est: Callable,
                        device="cpu"):
    """DFC-Nys combine over ranks (P/include/dfc/dfc.hpp:250-324, gen_nystrom
    P/include/dfc/sketch.hpp:241-266): subproblem 0 (C-hat = M[:, cols]) lives on rank 0 and
    subproblem 1 (R-hat = M[rows, :]) on rank shard(2, world, .)'s owner of block 1; R-hat's
    factors (d x k_R, n x k_R) are broadcast from that rank and rank 0 returns
    nystrom_fn(C_hat, make_est(R_left, R_right), rows, cols). None on the other ranks."""
    world, rank = dist.get_world_size(), dist.get_rank()
    src = 1 % world
    R = local_ests.get(1)
    rl = broadcast_array(dist, R.left if rank == src else None, src, device)
    rr = broadcast_array(dist, R.right if rank == src else None, src, device)
    if rank != 0:
        return None
    return nystrom_fn(local_ests[0], make_est(rl, rr), rows, cols)
