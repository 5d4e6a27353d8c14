"""TEST INFRASTRUCTURE ONLY — Python view of the CPU oracle (restated reference).

Loaded by tests/, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) as the checker / CPU baseline. The product package never
imports this module.  Parity status: pinned against the reference's RNG golden
vectors (P/tests/test_rng.cpp:11-48), its closed-form and exact-recovery unit
tests, and its printed acceptance values (P/test_output.txt:370-375) — see
tests/test_oracle_*.py.

Matrices cross the boundary column-major (Eigen layout, P/include/dfc/matrix_io.hpp:19);
this wrapper returns numpy arrays of the natural shape.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libdfc_oracle.so")

i64 = C.c_longlong
u64 = C.c_ulonglong
dptr = C.POINTER(C.c_double)
i64ptr = C.POINTER(C.c_longlong)
u64ptr = C.POINTER(C.c_ulonglong)


class OrcApgCfg(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("rel_tol", C.c_double), ("has_mu_init", C.c_int),
                ("mu_init", C.c_double), ("has_mu_floor", C.c_int), ("mu_floor", C.c_double),
                ("mu_decay", C.c_double), ("line_search", C.c_int)]


class OrcReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("objective", C.c_double), ("residual", C.c_double),
                ("rank", i64), ("wall_ms", C.c_double)]


class OrcTrace(C.Structure):
    _fields_ = [("it", C.c_int), ("rank", i64), ("k_final", i64), ("svd_calls", C.c_int),
                ("rel", C.c_double), ("mu", C.c_double), ("sigma_sum", C.c_double)]


class OrcDfcCfg(C.Structure):
    _fields_ = [("variant", C.c_int), ("ensemble", C.c_int), ("t", i64), ("l", i64), ("d", i64),
                ("rp_k", i64), ("rp_p", i64), ("rp_q", i64), ("seed", u64), ("solver", OrcApgCfg),
                ("task", C.c_int), ("lambda_", C.c_double), ("workers", C.c_int), ("ensemble_anchors", i64)]


class OrcDfcReport(C.Structure):
    _fields_ = [("divide_ms", C.c_double), ("factor_ms", C.c_double), ("combine_ms", C.c_double),
                ("total_ms", C.c_double), ("chosen_k", i64), ("k_clamped", C.c_int),
                ("rank_deficient", C.c_int), ("nsub", i64)]


class BlockError(RuntimeError):
    def __init__(self, block: int, msg: str):
        super().__init__(msg)
        self.block = block


_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (g++ + numpy's OpenBLAS)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = C.CDLL(_SO)
        L.orc_last_error.restype = C.c_char_p
        L.orc_last_error_block.restype = i64
        L.orc_factored_diff_norm.restype = C.c_double
        L.orc_default_rmf_lambda.restype = C.c_double
        L.orc_default_rmf_lambda.argtypes = [i64, i64]
        L.orc_trip_count.restype = i64
        # The reference solves each block single-threaded (Eigen without OpenMP,
        # P/CMakeLists.txt); parallelism comes only from DfcConfig.workers threads.
        L.orc_set_blas_threads(1)
        _lib = L
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    L = lib()
    msg = L.orc_last_error().decode()
    if rc == -1:
        raise ValueError(msg)
    if rc == -2:
        raise IndexError(msg)
    if rc == -3:
        raise BlockError(int(L.orc_last_error_block()), msg)
    raise RuntimeError(msg)


def _d(a):
    return a.ctypes.data_as(dptr)


def _i(a):
    return a.ctypes.data_as(i64ptr)


# ------------------------------------------------------------------ data model
@dataclass
class Observed:
    """ObservedMatrix (P/include/dfc/matrix_io.hpp:36-67): entries sorted column-major."""
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
    iterations: int
    objective: float
    residual: float
    rank: int
    wall_ms: float
    trace: list = field(default_factory=list)


class _Handle:
    def __init__(self, ptr, free):
        self.ptr, self._free = ptr, free

    def __del__(self):
        if self.ptr:
            self._free(self.ptr)
            self.ptr = None


def _obs_handle(obs: Observed):
    h = C.c_void_p()
    r = np.ascontiguousarray(obs.rows, dtype=np.int64)
    c = np.ascontiguousarray(obs.cols, dtype=np.int64)
    v = np.ascontiguousarray(obs.vals, dtype=np.float64)
    _check(lib().orc_obs_new(i64(obs.m), i64(obs.n), i64(len(v)), _i(r), _i(c), _d(v), C.byref(h)))
    return _Handle(h, lib().orc_obs_free)


def _obs_from_handle(h) -> Observed:
    L = lib()
    m, n, nnz = i64(), i64(), i64()
    L.orc_obs_dims(h, C.byref(m), C.byref(n), C.byref(nnz))
    r = np.empty(nnz.value, np.int64)
    c = np.empty(nnz.value, np.int64)
    v = np.empty(nnz.value, np.float64)
    L.orc_obs_get(h, _i(r), _i(c), _d(v))
    return Observed(m.value, n.value, r, c, v)


def _est_handle(e: Estimate):
    h = C.c_void_p()
    left = np.asfortranarray(e.left, dtype=np.float64)
    right = np.asfortranarray(e.right, dtype=np.float64)
    _check(lib().orc_est_new(i64(left.shape[0]), i64(right.shape[0]), i64(left.shape[1]),
                             _d(left), _d(right), C.byref(h)))
    return _Handle(h, lib().orc_est_free)


def _est_from_handle(h, free=True) -> Estimate:
    L = lib()
    m, n, k = i64(), i64(), i64()
    L.orc_est_dims(h, C.byref(m), C.byref(n), C.byref(k))
    left = np.empty((m.value, k.value), np.float64, order="F")
    right = np.empty((n.value, k.value), np.float64, order="F")
    L.orc_est_get(h, _d(left), _d(right))
    if free:
        L.orc_est_free(h)
    return Estimate(left, right)


def _trip_from_handle(h):
    L = lib()
    cnt = L.orc_trip_count(h)
    r = np.empty(cnt, np.int64)
    c = np.empty(cnt, np.int64)
    v = np.empty(cnt, np.float64)
    L.orc_trip_get(h, _i(r), _i(c), _d(v))
    L.orc_trip_free(h)
    return r, c, v


def make_observed(m, n, rows, cols, vals) -> Observed:
    """Validate and sort like the ObservedMatrix ctor (matrix_io.hpp:38-56)."""
    h = _obs_handle(Observed(m, n, np.asarray(rows), np.asarray(cols), np.asarray(vals)))
    return _obs_from_handle(h.ptr)


# ------------------------------------------------------------------ RNG / sampling
def rng_u64(seed, stream, n):
    out = np.empty(n, np.uint64)
    lib().orc_rng_u64(u64(seed), u64(stream), i64(n), out.ctypes.data_as(u64ptr))
    return out


def rng_uniform(seed, stream, n):
    out = np.empty(n, np.float64)
    lib().orc_rng_uniform(u64(seed), u64(stream), i64(n), _d(out))
    return out


def rng_uniform_pos(seed, stream, n):
    out = np.empty(n, np.float64)
    lib().orc_rng_uniform_pos(u64(seed), u64(stream), i64(n), _d(out))
    return out


def rng_normal(seed, stream, n):
    out = np.empty(n, np.float64)
    lib().orc_rng_normal(u64(seed), u64(stream), i64(n), _d(out))
    return out


def rng_index(seed, stream, count, bound):
    out = np.empty(count, np.uint64)
    _check(lib().orc_rng_index(u64(seed), u64(stream), i64(count), u64(bound), out.ctypes.data_as(u64ptr)))
    return out


def sample_without_replacement(seed, stream, n, l):
    out = np.empty(max(l, 0), np.int64)
    _check(lib().orc_sample_without_replacement(u64(seed), u64(stream), i64(n), i64(l), _i(out)))
    return out


def partition_columns(seed, stream, n, t):
    cols = np.empty(n, np.int64)
    offs = np.empty(max(t, 0) + 1, np.int64)
    _check(lib().orc_partition_columns(u64(seed), u64(stream), i64(n), i64(t), _i(cols), _i(offs)))
    return [cols[offs[g]:offs[g + 1]].copy() for g in range(t)]


def extract_columns(obs: Observed, idx) -> Observed:
    h = _obs_handle(obs)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = C.c_void_p()
    _check(lib().orc_extract_columns(h.ptr, i64(len(idx)), _i(idx), C.byref(out)))
    res = _obs_from_handle(out)
    lib().orc_obs_free(out)
    return res


def extract_rows(obs: Observed, idx) -> Observed:
    h = _obs_handle(obs)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = C.c_void_p()
    _check(lib().orc_extract_rows(h.ptr, i64(len(idx)), _i(idx), C.byref(out)))
    res = _obs_from_handle(out)
    lib().orc_obs_free(out)
    return res


# ------------------------------------------------------------------ generators
def gen_low_rank(m, n, r, seed, stream=0) -> Estimate:
    h = C.c_void_p()
    _check(lib().orc_gen_low_rank(i64(m), i64(n), i64(r), u64(seed), u64(stream), C.byref(h)))
    return _est_from_handle(h)


def gen_mc_instance(m, n, r, s, sigma, seed, stream=0):
    """gen_mc_instance (P/include/dfc/simgen.hpp:45-59) with SeededRng(seed, stream)."""
    hL, hO = C.c_void_p(), C.c_void_p()
    _check(lib().orc_gen_mc(i64(m), i64(n), i64(r), i64(s), C.c_double(sigma), u64(seed), u64(stream),
                            C.byref(hL), C.byref(hO)))
    obs = _obs_from_handle(hO)
    lib().orc_obs_free(hO)
    return _est_from_handle(hL), obs


def gen_rmf_instance(m, n, r, s, sigma, seed, stream=0, lo=0.0, hi=1.0):
    """gen_rmf_instance (simgen.hpp:64-82); lo/hi = outlier range (reference U[0,1])."""
    hL, hS = C.c_void_p(), C.c_void_p()
    M = np.empty((m, n), np.float64, order="F")
    _check(lib().orc_gen_rmf(i64(m), i64(n), i64(r), i64(s), C.c_double(sigma), u64(seed), u64(stream),
                             C.c_double(lo), C.c_double(hi), C.byref(hL), C.byref(hS), _d(M)))
    return _est_from_handle(hL), _trip_from_handle(hS), M


# ------------------------------------------------------------------ solvers
def apg_cfg(max_iters=500, rel_tol=1e-4, mu_init=None, mu_floor=None, mu_decay=0.7, line_search=False):
    return OrcApgCfg(max_iters, rel_tol, int(mu_init is not None), mu_init or 0.0,
                     int(mu_floor is not None), mu_floor or 0.0, mu_decay, int(line_search))


def high_accuracy():
    """ApgConfig::high_accuracy (P/include/dfc/solvers.hpp:29-36)."""
    return apg_cfg(max_iters=400, rel_tol=1e-9, mu_decay=0.5, mu_floor=0.0)


def _report(rep, tr, n):
    trace = [dict(it=tr[i].it, rank=tr[i].rank, k_final=tr[i].k_final, svd_calls=tr[i].svd_calls,
                  rel=tr[i].rel, mu=tr[i].mu, sigma_sum=tr[i].sigma_sum) for i in range(n)]
    return Report(rep.iterations, rep.objective, rep.residual, rep.rank, rep.wall_ms, trace)


def apg_mc(obs: Observed, cfg: OrcApgCfg | None = None):
    cfg = cfg or apg_cfg()
    h = _obs_handle(obs)
    out = C.c_void_p()
    rep = OrcReport()
    cap = cfg.max_iters
    tr = (OrcTrace * cap)()
    n = i64()
    _check(lib().orc_apg_mc(h.ptr, C.byref(cfg), C.byref(out), C.byref(rep), tr, i64(cap), C.byref(n)))
    return _est_from_handle(out), _report(rep, tr, min(n.value, cap))


def apg_rmf(M: np.ndarray, lam: float, cfg: OrcApgCfg | None = None):
    cfg = cfg or apg_cfg()
    M = np.asfortranarray(M, dtype=np.float64)
    hL, hS = C.c_void_p(), C.c_void_p()
    rep = OrcReport()
    cap = cfg.max_iters
    tr = (OrcTrace * cap)()
    n = i64()
    _check(lib().orc_apg_rmf(i64(M.shape[0]), i64(M.shape[1]), _d(M), C.c_double(lam), C.byref(cfg),
                             C.byref(hL), C.byref(hS), C.byref(rep), tr, i64(cap), C.byref(n)))
    return _est_from_handle(hL), _trip_from_handle(hS), _report(rep, tr, min(n.value, cap))


def default_rmf_lambda(m, n):
    return lib().orc_default_rmf_lambda(m, n)


def svt(A, tau) -> Estimate:
    A = np.asfortranarray(A, dtype=np.float64)
    out = C.c_void_p()
    _check(lib().orc_svt(i64(A.shape[0]), i64(A.shape[1]), _d(A), C.c_double(tau), C.byref(out)))
    return _est_from_handle(out)


def soft_threshold(A, tau):
    A = np.asfortranarray(A, dtype=np.float64)
    out = np.empty_like(A, order="F")
    _check(lib().orc_soft_threshold(i64(A.shape[0]), i64(A.shape[1]), _d(A), C.c_double(tau), _d(out)))
    return out


def compact_svd_estimate(A) -> Estimate:
    A = np.asfortranarray(A, dtype=np.float64)
    out = C.c_void_p()
    _check(lib().orc_compact_svd(i64(A.shape[0]), i64(A.shape[1]), _d(A), C.byref(out)))
    return _est_from_handle(out)


def factored_diff_norm(a: Estimate, b: Estimate) -> float:
    ha, hb = _est_handle(a), _est_handle(b)
    return lib().orc_factored_diff_norm(ha.ptr, hb.ptr)


def rmse(truth: Estimate, est: Estimate) -> float:
    """rmse (P/include/dfc/bench.hpp:80-86): factored diff norm / sqrt(cells)."""
    m, n = truth.left.shape[0], truth.right.shape[0]
    return factored_diff_norm(truth, est) / np.sqrt(float(m) * float(n))


# ------------------------------------------------------------------ combiners
def _plan_arrays(groups):
    offs = np.zeros(len(groups) + 1, np.int64)
    offs[1:] = np.cumsum([len(g) for g in groups])
    cols = np.ascontiguousarray(np.concatenate([np.asarray(g, np.int64) for g in groups]), np.int64)
    return offs, cols


def _est_array(ests):
    hs = [_est_handle(e) for e in ests]
    arr = (C.c_void_p * len(hs))(*[h.ptr for h in hs])
    return hs, arr


def column_project(basis: Estimate, blocks, groups) -> Estimate:
    hb = _est_handle(basis)
    hs, arr = _est_array(blocks)
    offs, cols = _plan_arrays(groups)
    out = C.c_void_p()
    _check(lib().orc_column_project(hb.ptr, i64(len(blocks)), arr, _i(offs), _i(cols), i64(len(cols)),
                                    C.byref(out)))
    return _est_from_handle(out)


def random_project(blocks, groups, k, p, q, seed, stream) -> Estimate:
    hs, arr = _est_array(blocks)
    offs, cols = _plan_arrays(groups)
    out = C.c_void_p()
    _check(lib().orc_random_project(i64(len(blocks)), arr, _i(offs), _i(cols), i64(len(cols)), i64(k), i64(p),
                                    i64(q), u64(seed), u64(stream), C.byref(out)))
    return _est_from_handle(out)


def gen_nystrom(C_hat: Estimate, R_hat: Estimate, rows, cols) -> Estimate:
    hc, hr = _est_handle(C_hat), _est_handle(R_hat)
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    out = C.c_void_p()
    _check(lib().orc_gen_nystrom(hc.ptr, hr.ptr, i64(len(rows)), _i(rows), i64(len(cols)), _i(cols),
                                 C.byref(out)))
    return _est_from_handle(out)


def average_estimates(ests, recompress_to=None) -> Estimate:
    hs, arr = _est_array(ests)
    out = C.c_void_p()
    _check(lib().orc_average_estimates(i64(len(ests)), arr, i64(-1 if recompress_to is None else recompress_to),
                                       C.byref(out)))
    return _est_from_handle(out)


# ------------------------------------------------------------------ orchestrator
VARIANTS = {"proj": 0, "rp": 1, "nys": 2}
TASKS = {"mc": 0, "rmf": 1}


def dfc_run(obs: Observed, variant="proj", ensemble=False, t=4, l=0, d=0, rp_p=5, rp_q=2, seed=0,
            solver_cfg: OrcApgCfg | None = None, task="mc", lam=0.0, workers=1, ensemble_anchors=0):
    """dfc_run (P/include/dfc/dfc.hpp:326-335) with the reference's DfcConfig fields."""
    cfg = OrcDfcCfg(VARIANTS[variant], int(ensemble), t, l, d, 1, rp_p, rp_q, seed,
                    solver_cfg or apg_cfg(), TASKS[task], lam, workers, ensemble_anchors)
    h = _obs_handle(obs)
    out = C.c_void_p()
    rep = OrcDfcReport()
    subs = (OrcReport * 4096)()
    _check(lib().orc_dfc_run(h.ptr, C.byref(cfg), C.byref(out), C.byref(rep), subs, i64(4096)))
    est = _est_from_handle(out)
    sub = [Report(subs[i].iterations, subs[i].objective, subs[i].residual, subs[i].rank, subs[i].wall_ms)
           for i in range(min(rep.nsub, 4096))]
    return est, dict(divide_ms=rep.divide_ms, factor_ms=rep.factor_ms, combine_ms=rep.combine_ms,
                     total_ms=rep.total_ms, chosen_k=rep.chosen_k, k_clamped=bool(rep.k_clamped),
                     rank_deficient=bool(rep.rank_deficient), subproblems=sub)


class McRun:
    """Resumable apg_mc (orc_mc_run_*): step(n) -> per-iteration trace; finish() -> (Estimate,
    Report) of the current iterate without ending the run (bench windows, fixture generation)."""

    def __init__(self, obs: Observed, cfg: OrcApgCfg | None = None):
        self._h = _obs_handle(obs)
        self.ptr = C.c_void_p()
        _check(lib().orc_mc_run_new(self._h.ptr, C.byref(cfg or apg_cfg()), C.byref(self.ptr)))

    def step(self, n: int):
        tr = (OrcTrace * max(n, 1))()
        done, ln = i64(), i64()
        _check(lib().orc_mc_run_step_trace(self.ptr, i64(n), C.byref(done), tr, i64(max(n, 1)), C.byref(ln)))
        return _report(OrcReport(), tr, min(ln.value, max(n, 1))).trace

    def finish(self):
        out = C.c_void_p()
        rep = OrcReport()
        _check(lib().orc_mc_run_finish(self.ptr, C.byref(out), C.byref(rep)))
        return _est_from_handle(out), _report(rep, None, 0)

    def close(self):
        if self.ptr:
            lib().orc_mc_run_free(self.ptr)
            self.ptr = None

    def __del__(self):
        self.close()
