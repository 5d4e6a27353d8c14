"""Multi-GPU DFC (one process per GPU) over libdfcg's native distributed path.

The sharding, the LPT assignment and the combine's exchanges all live in the C++ library
(csrc/dfc_dist.cpp, csrc/dist.cpp; C ABI ``dfcg_dfc_run_dist``): every rank passes the same
observations and DfcConfig, solves its LPT share of the subproblems with no exchange during the
solve (P/include/dfc/dfc.hpp:133-147: they are independent), and the combine moves factors only
— the basis U_b broadcast and the projected-row gather for DFC-Proj (sketch.hpp:170-199), R-hat's
factors for DFC-Nys (sketch.hpp:241-266), the block factors for DFC-RP.

This module is the torch.distributed plumbing around it:
  Comm.nccl(...)  NCCL communicator inside libdfcg (NVLink / NVSwitch); the ncclUniqueId is drawn
                  on rank 0 and broadcast over the caller's process group;
  Comm.host(...)  the library's host-callback transport driven by torch.distributed collectives on
                  CPU tensors (gloo) — the CPU test transport, and a fallback without NCCL.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence

import numpy as np

from . import _lib as L

_BCAST = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32)
_SEND = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32)
_RECV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32)


class HostTransportC(C.Structure):
    _fields_ = [("user", C.c_void_p), ("bcast", _BCAST), ("send", _SEND), ("recv", _RECV)]


def assign_blocks(nnz: Sequence[int], nranks: int) -> List[int]:
    """LPT owner of every subproblem (dfcg_assign_blocks): descending nnz, each to the
    least-loaded rank. Pure host code (works without a GPU)."""
    a = np.ascontiguousarray(np.asarray(nnz, dtype=np.int64))
    out = np.zeros(len(a), np.int32)
    L._check(L.lib().dfcg_assign_blocks(C.c_int64(len(a)), a.ctypes.data_as(L.i64ptr), C.c_int32(nranks),
                                        out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out.tolist()


def _host_view(buf, nbytes):
    import torch

    arr = np.ctypeslib.as_array((C.c_uint8 * int(nbytes)).from_address(buf))
    return torch.from_numpy(arr)


class Comm:
    """dfcg_comm handle (see module docstring)."""

    def __init__(self, handle: C.c_void_p, rank: int, size: int, keep=()):
        self._h, self.rank, self.size, self._keep = handle, rank, size, keep

    @classmethod
    def nccl(cls, group=None, device: int = 0) -> "Comm":
        import torch
        import torch.distributed as dist

        rank, size = dist.get_rank(group), dist.get_world_size(group)
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            L._check(L.lib().dfcg_nccl_unique_id(uid))
        dev = f"cuda:{device}" if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=dev)
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (C.c_ubyte * 128)(*t.cpu().tolist())
        h = C.c_void_p()
        L._check(L.lib().dfcg_comm_init_nccl(L.context(device), C.c_int32(size), C.c_int32(rank), uid, C.byref(h)))
        return cls(h, rank, size)

    @classmethod
    def host(cls, group=None) -> "Comm":
        import torch.distributed as dist

        rank, size = dist.get_rank(group), dist.get_world_size(group)

        def glob(r):
            return dist.get_global_rank(group, r) if group is not None else r

        def bcast(user, buf, nbytes, root):
            try:
                dist.broadcast(_host_view(buf, nbytes), src=glob(root), group=group)
                return 0
            except Exception:  # noqa: BLE001 — reported to the library as a transport failure
                return 1

        def send(user, buf, nbytes, peer):
            try:
                dist.send(_host_view(buf, nbytes), dst=glob(peer), group=group)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        def recv(user, buf, nbytes, peer):
            try:
                dist.recv(_host_view(buf, nbytes), src=glob(peer), group=group)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        cb = (_BCAST(bcast), _SEND(send), _RECV(recv))
        tr = HostTransportC(None, *cb)
        h = C.c_void_p()
        L._check(L.lib().dfcg_comm_init_host(C.c_int32(size), C.c_int32(rank), C.byref(tr), C.byref(h)))
        return cls(h, rank, size, keep=(cb, tr))

    def selftest(self) -> int:
        """Host-only traffic through the transport; returns the mismatched words this rank saw."""
        err = C.c_int64()
        L._check(L.lib().dfcg_comm_selftest(self._h, C.byref(err)))
        return err.value

    def close(self):
        if self._h:
            L.lib().dfcg_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def dfc_run_dist(obs: L.Observed, comm: Comm, variant="proj", ensemble=False, t=4, l=0, d=0, rp_p=5, rp_q=2,
                 seed=0, solver_cfg: L.ApgConfig | None = None, task="mc", lam=0.0, workers=1, device: int = 0,
                 ensemble_anchors: int = 0):
    """dfc_run over the ranks of `comm` (dfcg_dfc_run_dist): same arguments and result as
    paper_1107_0789_b200.dfc_run on every rank; info adds the LPT `owner` of every subproblem."""
    keep = L._Keep()
    o = L._obs_in(obs, keep)
    cfg = L.DfcCfgC(L.VARIANTS[variant], int(ensemble), t, l, d, rp_p, rp_q, seed, (solver_cfg or L.ApgConfig()).c(),
                    L.TASKS[task], lam, workers, ensemble_anchors)
    out = L.LowRankC()
    rep = L.DfcReportC()
    owner = (C.c_int32 * 4096)()
    L._check(L.lib().dfcg_dfc_run_dist(L.context(device), comm._h, C.byref(o), C.byref(cfg), C.byref(out),
                                       C.byref(rep), owner, C.c_int64(4096)))
    subs = [L.Report(rep.subproblems[i].iterations, rep.subproblems[i].objective, rep.subproblems[i].residual,
                     rep.subproblems[i].rank, rep.subproblems[i].wall_ms) for i in range(rep.n_sub)]
    info = dict(divide_ms=rep.divide_ms, factor_ms=rep.factor_ms, combine_ms=rep.combine_ms,
                total_ms=rep.total_ms, chosen_k=rep.chosen_k, k_clamped=bool(rep.k_clamped),
                rank_deficient=bool(rep.rank_deficient), subproblems=subs,
                owner=[owner[i] for i in range(min(rep.n_sub, 4096))])
    L.lib().dfcg_dfc_report_free(C.byref(rep))
    return L._lowrank_out(out), info
