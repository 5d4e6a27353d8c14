"""ctypes binding of libdfcg.so (include/dfcg.h).

Mirrors the reference's operator interface (P/include/dfc/solvers.hpp, sketch.hpp, dfc.hpp):
same names, same argument meaning, same exceptions (ValueError for std::invalid_argument,
IndexError for std::out_of_range, BlockError for dfc::BlockError). Matrices are numpy arrays
of their natural shape; they cross the ABI column-major, as Eigen stores them.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_PKG, "_lib", "libdfcg.so")
_CSRC = os.path.join(_PKG, "csrc")

i64 = C.c_int64
u64 = C.c_uint64
dptr = C.POINTER(C.c_double)
i64ptr = C.POINTER(C.c_int64)


class DfcError(RuntimeError):
    """CUDA / internal failure inside libdfcg (DFCG_ECUDA, DFCG_ENOMEM, DFCG_EINTERNAL)."""


class BlockError(RuntimeError):
    """dfc::BlockError (P/include/dfc/dfc.hpp:50-54): lowest failing block index + message."""

    def __init__(self, block: int, msg: str):
        super().__init__(f"block {block}: {msg}")  # the reference's what() (dfc.hpp:51-52)
        self.block = block
        self.inner = msg


class ApgCfgC(C.Structure):
    _fields_ = [("max_iters", C.c_int32), ("rel_tol", C.c_double), ("has_mu_init", C.c_int32),
                ("mu_init", C.c_double), ("has_mu_floor", C.c_int32), ("mu_floor", C.c_double),
                ("mu_decay", C.c_double), ("line_search", C.c_int32)]


class ReportC(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("objective", C.c_double), ("residual", C.c_double),
                ("rank", i64), ("wall_ms", C.c_double)]


class ObsC(C.Structure):
    _fields_ = [("m", i64), ("n", i64), ("nnz", i64), ("row", i64ptr), ("col", i64ptr), ("val", dptr)]


class LowRankC(C.Structure):
    _fields_ = [("m", i64), ("n", i64), ("k", i64), ("left", dptr), ("right", dptr)]


class SparseC(C.Structure):
    _fields_ = [("m", i64), ("n", i64), ("count", i64), ("row", i64ptr), ("col", i64ptr), ("val", dptr)]


class TraceC(C.Structure):
    _fields_ = [("it", C.c_int32), ("rank", i64), ("k_final", i64), ("svd_calls", C.c_int32),
                ("rel", C.c_double), ("mu", C.c_double), ("sigma_sum", C.c_double), ("ms", C.c_double)]


class DfcCfgC(C.Structure):
    _fields_ = [("variant", C.c_int32), ("ensemble", C.c_int32), ("t", i64), ("l", i64), ("d", i64),
                ("rp_p", i64), ("rp_q", i64), ("seed", u64), ("solver", ApgCfgC), ("task", C.c_int32),
                ("lambda_", C.c_double), ("workers", C.c_int32), ("ensemble_anchors", i64)]


class DfcReportC(C.Structure):
    _fields_ = [("divide_ms", C.c_double), ("factor_ms", C.c_double), ("combine_ms", C.c_double),
                ("total_ms", C.c_double), ("chosen_k", i64), ("k_clamped", C.c_int32),
                ("rank_deficient", C.c_int32), ("n_sub", i64), ("subproblems", C.POINTER(ReportC))]


# ------------------------------------------------------------------ library loading
_lib = None
_lock = threading.Lock()


def lib_path() -> str:
    return _SO


def build() -> str:
    """Compile libdfcg.so in-tree for sm_100a (nvcc; see csrc/Makefile)."""
    subprocess.run(["make", "-s", "-C", _CSRC, "-j8"], check=True)
    return _SO


def lib():
    """Load libdfcg.so. Raises (no fallback) if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_SO):
                raise DfcError(f"libdfcg.so not built ({_SO}); run paper_1107_0789_b200.build()")
            L = C.CDLL(_SO)
            L.dfcg_last_error.restype = C.c_char_p
            L.dfcg_last_error_block.restype = i64
            L.dfcg_last_error_line.restype = i64
            _lib = L
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    L = lib()
    msg = L.dfcg_last_error().decode()
    if rc == -1:
        raise ValueError(msg)
    if rc == -2:
        raise IndexError(msg)
    if rc == -3:
        raise BlockError(int(L.dfcg_last_error_block()), msg)
    if rc == -8:
        raise ParseError(int(L.dfcg_last_error_line()), msg)
    raise DfcError(f"libdfcg error {rc}: {msg}")


_contexts: dict[int, C.c_void_p] = {}


def context(device: int = 0) -> C.c_void_p:
    """Per-process dfcg_ctx for a CUDA device (created on first use)."""
    with _lock:
        ctx = _contexts.get(device)
    if ctx is None:
        h = C.c_void_p()
        _check(lib().dfcg_ctx_create(C.c_int(device), C.byref(h)))
        with _lock:
            _contexts[device] = h
        ctx = h
    return ctx


class ParseError(RuntimeError):
    """dfc::ParseError (P/include/dfc/matrix_io.hpp:22-26): "line N: what", with .line."""

    def __init__(self, line: int, msg: str):
        super().__init__(msg)  # libdfcg's message already carries the "line N: " prefix
        self.line = line


# ------------------------------------------------------------------ data model
@dataclass
class Observed:
    """ObservedMatrix (P/include/dfc/matrix_io.hpp:36-67)."""
    m: int
    n: int
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray

    @property
    def count(self):
        return len(self.vals)


@dataclass
class Estimate:
    """LowRankEstimate (matrix_io.hpp:71-98): L = left @ right.T."""
    left: np.ndarray
    right: np.ndarray

    @property
    def rank(self):
        return self.left.shape[1]

    def dense(self):
        return self.left @ self.right.T


@dataclass
class Report:
    """SolveReport (P/include/dfc/solvers.hpp:39-45) + per-iteration trace."""
    iterations: int
    objective: float
    residual: float
    rank: int
    wall_ms: float
    trace: list = field(default_factory=list)


@dataclass
class ApgConfig:
    """ApgConfig (P/include/dfc/solvers.hpp:19-37)."""
    max_iters: int = 500
    rel_tol: float = 1e-4
    mu_init: float | None = None
    mu_floor: float | None = None
    mu_decay: float = 0.7
    line_search: bool = False

    def c(self) -> ApgCfgC:
        return ApgCfgC(self.max_iters, self.rel_tol, int(self.mu_init is not None), self.mu_init or 0.0,
                       int(self.mu_floor is not None), self.mu_floor or 0.0, self.mu_decay,
                       int(self.line_search))


def high_accuracy() -> ApgConfig:
    """ApgConfig::high_accuracy (P/include/dfc/solvers.hpp:29-36)."""
    return ApgConfig(max_iters=400, rel_tol=1e-9, mu_decay=0.5, mu_floor=0.0)


def _d(a):
    return a.ctypes.data_as(dptr)


def _i(a):
    return a.ctypes.data_as(i64ptr)


class _Keep:
    """Holds numpy buffers alive while a ctypes struct points into them."""

    def __init__(self):
        self.refs = []

    def f(self, a):
        a = np.asfortranarray(a, dtype=np.float64)
        self.refs.append(a)
        return a

    def i(self, a):
        a = np.ascontiguousarray(a, dtype=np.int64)
        self.refs.append(a)
        return a


def _lowrank_in(e: Estimate, keep: _Keep) -> LowRankC:
    left = keep.f(e.left)
    right = keep.f(e.right)
    if left.ndim != 2 or right.ndim != 2:
        raise ValueError("LowRankEstimate: factors must be 2-D")
    return LowRankC(left.shape[0], right.shape[0], left.shape[1], _d(left), _d(right))


def _lowrank_out(c: LowRankC) -> Estimate:
    m, n, k = c.m, c.n, c.k
    if k == 0:
        lib().dfcg_lowrank_free(C.byref(c))
        return Estimate(np.zeros((m, 0), order="F"), np.zeros((n, 0), order="F"))
    left = np.ctypeslib.as_array(c.left, shape=(max(k, 1) * m,))[: m * k].copy().reshape((m, k), order="F")
    right = np.ctypeslib.as_array(c.right, shape=(max(k, 1) * n,))[: n * k].copy().reshape((n, k), order="F")
    lib().dfcg_lowrank_free(C.byref(c))
    return Estimate(left, right)


def _obs_in(obs: Observed, keep: _Keep) -> ObsC:
    r, c = keep.i(obs.rows), keep.i(obs.cols)
    v = np.ascontiguousarray(obs.vals, dtype=np.float64)
    keep.refs.append(v)
    if not (len(r) == len(c) == len(v)):
        raise ValueError("ObservedMatrix: ragged triplets")
    return ObsC(obs.m, obs.n, len(v), _i(r), _i(c), _d(v))


def _trace_list(tr, n):
    return [dict(it=tr[i].it, rank=tr[i].rank, k_final=tr[i].k_final, svd_calls=tr[i].svd_calls, rel=tr[i].rel,
                 mu=tr[i].mu, sigma_sum=tr[i].sigma_sum, ms=tr[i].ms) for i in range(n)]


# ------------------------------------------------------------------ F step
def apg_mc(obs: Observed, cfg: ApgConfig | None = None, device: int = 0):
    """apg_mc (P/include/dfc/solvers.hpp:241-327) on the GPU. Returns (Estimate, Report)."""
    cfg = cfg or ApgConfig()
    keep = _Keep()
    o = _obs_in(obs, keep)
    out = LowRankC()
    rep = ReportC()
    cap = max(cfg.max_iters, 1)
    tr = (TraceC * cap)()
    n = i64()
    _check(lib().dfcg_apg_mc(context(device), C.byref(o), C.byref(cfg.c()), C.byref(out), C.byref(rep), tr,
                             i64(cap), C.byref(n)))
    return _lowrank_out(out), Report(rep.iterations, rep.objective, rep.residual, rep.rank, rep.wall_ms,
                                     _trace_list(tr, min(n.value, cap)))


def apg_rmf(M: np.ndarray, lam: float, cfg: ApgConfig | None = None, device: int = 0):
    """apg_rmf (solvers.hpp:332-414). Returns (Estimate, (rows, cols, vals) of S_hat, Report)."""
    cfg = cfg or ApgConfig()
    M = np.asfortranarray(M, dtype=np.float64)
    L = LowRankC()
    S = SparseC()
    rep = ReportC()
    cap = max(cfg.max_iters, 1)
    tr = (TraceC * cap)()
    n = i64()
    _check(lib().dfcg_apg_rmf(context(device), _d(M), i64(M.shape[0]), i64(M.shape[1]), C.c_double(lam),
                              C.byref(cfg.c()), C.byref(L), C.byref(S), C.byref(rep), tr, i64(cap), C.byref(n)))
    cnt = S.count
    rows = np.ctypeslib.as_array(S.row, shape=(max(cnt, 1),))[:cnt].copy()
    cols = np.ctypeslib.as_array(S.col, shape=(max(cnt, 1),))[:cnt].copy()
    vals = np.ctypeslib.as_array(S.val, shape=(max(cnt, 1),))[:cnt].copy()
    lib().dfcg_sparse_free(C.byref(S))
    return _lowrank_out(L), (rows, cols, vals), Report(rep.iterations, rep.objective, rep.residual, rep.rank,
                                                       rep.wall_ms, _trace_list(tr, min(n.value, cap)))


class McSolver:
    """Resumable apg_mc with Omega resident on the GPU (dfcg_mc_solver_*)."""

    def __init__(self, obs: Observed, cfg: ApgConfig | None = None, device: int = 0):
        self.cfg = cfg or ApgConfig()
        keep = _Keep()
        o = _obs_in(obs, keep)
        self._h = C.c_void_p()
        _check(lib().dfcg_mc_solver_create(context(device), C.byref(o), C.byref(self.cfg.c()), C.byref(self._h)))

    def step(self, n: int = 1, trace: bool = False):
        done = i64()
        cap = max(n, 1) if trace else 0
        tr = (TraceC * max(cap, 1))()
        tl = i64()
        _check(lib().dfcg_mc_solver_step(self._h, i64(n), C.byref(done), tr if trace else None, i64(cap),
                                         C.byref(tl)))
        return (done.value, _trace_list(tr, min(tl.value, cap))) if trace else done.value

    def finish(self):
        out = LowRankC()
        rep = ReportC()
        _check(lib().dfcg_mc_solver_finish(self._h, C.byref(out), C.byref(rep)))
        return _lowrank_out(out), Report(rep.iterations, rep.objective, rep.residual, rep.rank, rep.wall_ms)

    def close(self):
        if self._h:
            lib().dfcg_mc_solver_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ C step
def _plan(groups, keep):
    offs = np.zeros(len(groups) + 1, np.int64)
    offs[1:] = np.cumsum([len(g) for g in groups])
    cols = np.concatenate([np.asarray(g, np.int64) for g in groups]) if groups else np.zeros(0, np.int64)
    return keep.i(offs), keep.i(cols)


def column_project(basis: Estimate, blocks, groups, device: int = 0) -> Estimate:
    """column_project (P/include/dfc/sketch.hpp:170-199)."""
    keep = _Keep()
    b = _lowrank_in(basis, keep)
    arr = (LowRankC * max(len(blocks), 1))(*[_lowrank_in(e, keep) for e in blocks])
    offs, cols = _plan(groups, keep)
    out = LowRankC()
    _check(lib().dfcg_column_project(context(device), C.byref(b), i64(len(blocks)), arr, _i(offs), _i(cols),
                                     i64(len(cols)), C.byref(out)))
    return _lowrank_out(out)


def gen_nystrom(C_hat: Estimate, R_hat: Estimate, rows, cols, device: int = 0) -> Estimate:
    """gen_nystrom (sketch.hpp:241-266)."""
    keep = _Keep()
    c = _lowrank_in(C_hat, keep)
    r = _lowrank_in(R_hat, keep)
    ri, ci = keep.i(rows), keep.i(cols)
    out = LowRankC()
    _check(lib().dfcg_gen_nystrom(context(device), C.byref(c), C.byref(r), i64(len(ri)), _i(ri), i64(len(ci)),
                                  _i(ci), C.byref(out)))
    return _lowrank_out(out)


def average_estimates(ests, recompress_to=None, device: int = 0) -> Estimate:
    """average_estimates (sketch.hpp:271-298)."""
    keep = _Keep()
    arr = (LowRankC * max(len(ests), 1))(*[_lowrank_in(e, keep) for e in ests])
    out = LowRankC()
    _check(lib().dfcg_average_estimates(context(device), i64(len(ests)), arr,
                                        i64(-1 if recompress_to is None else recompress_to), C.byref(out)))
    return _lowrank_out(out)


def random_project(blocks, groups, k, p, q, seed, stream, device: int = 0) -> Estimate:
    """random_project (sketch.hpp:204-237) with SeededRng(seed, stream)."""
    keep = _Keep()
    arr = (LowRankC * max(len(blocks), 1))(*[_lowrank_in(e, keep) for e in blocks])
    offs, cols = _plan(groups, keep)
    out = LowRankC()
    _check(lib().dfcg_random_project(context(device), i64(len(blocks)), arr, _i(offs), _i(cols), i64(len(cols)),
                                     i64(k), i64(p), i64(q), u64(seed), u64(stream), C.byref(out)))
    return _lowrank_out(out)


def svd_of_product(left: np.ndarray, right: np.ndarray, device: int = 0):
    """svd_of_product (sketch.hpp:73-86). Returns (Estimate (U, V diag s), s)."""
    keep = _Keep()
    left = keep.f(left)
    right = keep.f(right)
    if left.shape[1] != right.shape[1]:
        raise ValueError("svd_of_product: rank mismatch")
    inp = LowRankC(left.shape[0], right.shape[0], left.shape[1], _d(left), _d(right))
    s = np.zeros(max(1, min(left.shape[0], right.shape[0], left.shape[1])), np.float64)
    out = LowRankC()
    r = i64()
    _check(lib().dfcg_svd_of_product(context(device), C.byref(inp), C.byref(out), _d(s), C.byref(r)))
    return _lowrank_out(out), s[: r.value].copy()


def project_block(Ub: np.ndarray, block: Estimate, device: int = 0) -> np.ndarray:
    """One block of column_project (P/include/dfc/sketch.hpp:194-196): right_g (Ub^T left_g)^T."""
    keep = _Keep()
    U = keep.f(Ub)
    b = _lowrank_in(block, keep)
    out = np.empty((block.right.shape[0], U.shape[1]), np.float64, order="F")
    _check(lib().dfcg_project_block(context(device), _d(U), i64(U.shape[0]), i64(U.shape[1]), C.byref(b), _d(out)))
    return out


VARIANTS = {"proj": 0, "rp": 1, "nys": 2}
TASKS = {"mc": 0, "rmf": 1}


def dfc_run(obs: Observed, variant="proj", ensemble=False, t=4, l=0, d=0, rp_p=5, rp_q=2, seed=0,
            solver_cfg: ApgConfig | None = None, task="mc", lam=0.0, workers=1, device: int = 0,
            ensemble_anchors: int = 0):
    """dfc_run (P/include/dfc/dfc.hpp:326-335): D on host, F and C on the GPU. ensemble_anchors
    (Proj-Ens only): 0 = every block anchors the ensemble, as in the reference; A > 0 = the first
    min(A, t) plan groups (BASELINE c5's "ensemble of 4")."""
    keep = _Keep()
    o = _obs_in(obs, keep)
    cfg = DfcCfgC(VARIANTS[variant], int(ensemble), t, l, d, rp_p, rp_q, seed, (solver_cfg or ApgConfig()).c(),
                  TASKS[task], lam, workers, ensemble_anchors)
    out = LowRankC()
    rep = DfcReportC()
    _check(lib().dfcg_dfc_run(context(device), C.byref(o), C.byref(cfg), C.byref(out), C.byref(rep)))
    subs = [Report(rep.subproblems[i].iterations, rep.subproblems[i].objective, rep.subproblems[i].residual,
                   rep.subproblems[i].rank, rep.subproblems[i].wall_ms) for i in range(rep.n_sub)]
    info = dict(divide_ms=rep.divide_ms, factor_ms=rep.factor_ms, combine_ms=rep.combine_ms,
                total_ms=rep.total_ms, chosen_k=rep.chosen_k, k_clamped=bool(rep.k_clamped),
                rank_deficient=bool(rep.rank_deficient), subproblems=subs)
    lib().dfcg_dfc_report_free(C.byref(rep))
    return _lowrank_out(out), info
