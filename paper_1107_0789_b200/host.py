"""Host utilities of libdfcg.so (include/dfcg_host.h): the reference's SeededRng, sampling
and instance generators (P/include/dfc/rng.hpp, sampling.hpp, simgen.hpp), in C++.

These build the exact inputs the reference builds (same seeds, same draw order); they do not
touch the GPU and are what bench.py uses to synthesise its workloads.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import Estimate, LowRankC, Observed, SparseC, _check, _d, _i, _lowrank_out, i64, i64ptr, lib, u64

dpp = C.POINTER(C.POINTER(C.c_double))


class SeededRng:
    """Stateless view: draws the first n values of SeededRng(seed, stream)."""

    def __init__(self, seed: int, stream: int = 0):
        self.seed, self.stream = seed, stream

    def u64(self, n):
        out = np.empty(n, np.uint64)
        lib().dfcg_rng_u64(u64(self.seed), u64(self.stream), i64(n), out.ctypes.data_as(C.POINTER(C.c_uint64)))
        return out

    def uniform(self, n):
        out = np.empty(n, np.float64)
        lib().dfcg_rng_uniform(u64(self.seed), u64(self.stream), i64(n), _d(out))
        return out

    def normal(self, n):
        out = np.empty(n, np.float64)
        lib().dfcg_rng_normal(u64(self.seed), u64(self.stream), i64(n), _d(out))
        return out

    def index(self, count, bound):
        out = np.empty(count, np.uint64)
        _check(lib().dfcg_rng_index(u64(self.seed), u64(self.stream), i64(count), u64(bound),
                                    out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out


def sample_without_replacement(seed, stream, n, l):
    out = np.empty(max(l, 0), np.int64)
    _check(lib().dfcg_sample_without_replacement(u64(seed), u64(stream), i64(n), i64(l), _i(out)))
    return out


def partition_columns(seed, stream, n, t):
    cols = np.empty(max(n, 0), np.int64)
    offs = np.empty(max(t, 0) + 1, np.int64)
    _check(lib().dfcg_partition_columns(u64(seed), u64(stream), i64(n), i64(t), _i(cols), _i(offs)))
    return [cols[offs[g]:offs[g + 1]].copy() for g in range(t)]


def extract_subproblems(obs: Observed, groups, rows=None):
    """libdfcg's D step (dfcg_extract_subproblems): the column groups, then the row sample, in
    one parallel pass — what dfc_run extracts (P/include/dfc/sampling.hpp:83-113)."""
    from ._lib import ObsC, _Keep, _obs_in

    keep = _Keep()
    o = _obs_in(obs, keep)
    offs = np.zeros(len(groups) + 1, np.int64)
    offs[1:] = np.cumsum([len(g) for g in groups])
    cols = np.ascontiguousarray(np.concatenate([np.asarray(g, np.int64) for g in groups]) if groups else
                                np.zeros(1, np.int64))
    rr = np.ascontiguousarray(np.asarray(rows if rows is not None else [0], np.int64))
    nsub = len(groups) + (rows is not None)
    counts = np.zeros(max(nsub, 1), np.int64)
    pr, pc, pv = i64ptr(), i64ptr(), C.POINTER(C.c_double)()
    _check(lib().dfcg_extract_subproblems(C.byref(o), i64(len(groups)), _i(offs), _i(cols),
                                          i64(len(rows) if rows is not None else 0), _i(rr), _i(counts),
                                          C.byref(pr), C.byref(pc), C.byref(pv)))
    total = int(counts[:nsub].sum())
    R = np.ctypeslib.as_array(pr, (max(total, 1),))[:total].copy()
    Cc = np.ctypeslib.as_array(pc, (max(total, 1),))[:total].copy()
    V = np.ctypeslib.as_array(pv, (max(total, 1),))[:total].copy()
    for p in (pr, pc, pv):
        lib().dfcg_free(p)
    out, at = [], 0
    for i in range(nsub):
        c = int(counts[i])
        is_row = rows is not None and i == nsub - 1
        m = len(rows) if is_row else obs.m
        n = obs.n if is_row else len(groups[i])
        out.append(Observed(m, n, R[at:at + c], Cc[at:at + c], V[at:at + c]))
        at += c
    return out


def extract_columns(obs: Observed, idx) -> Observed:
    """extract_columns (P/include/dfc/sampling.hpp:83-97), vectorised."""
    idx = np.asarray(idx, np.int64)
    pos = np.full(obs.n, -1, np.int64)
    if np.any((idx < 0) | (idx >= obs.n)):
        raise IndexError("extract_columns: index out of range")
    if len(np.unique(idx)) != len(idx):
        raise ValueError("extract_columns: duplicate index")
    pos[idx] = np.arange(len(idx))
    p = pos[obs.cols]
    keep = p >= 0
    r, c, v = obs.rows[keep], p[keep], obs.vals[keep]
    order = np.lexsort((r, c))
    return Observed(obs.m, len(idx), r[order], c[order], v[order])


def extract_rows(obs: Observed, idx) -> Observed:
    """extract_rows (sampling.hpp:99-113), vectorised."""
    idx = np.asarray(idx, np.int64)
    pos = np.full(obs.m, -1, np.int64)
    if np.any((idx < 0) | (idx >= obs.m)):
        raise IndexError("extract_rows: index out of range")
    if len(np.unique(idx)) != len(idx):
        raise ValueError("extract_rows: duplicate index")
    pos[idx] = np.arange(len(idx))
    p = pos[obs.rows]
    keep = p >= 0
    r, c, v = p[keep], obs.cols[keep], obs.vals[keep]
    order = np.lexsort((r, c))
    return Observed(len(idx), obs.n, r[order], c[order], v[order])


def median_rank(ranks):
    """median_rank (P/include/dfc/dfc.hpp:159-164): lower median floored at 1."""
    if len(ranks) == 0:
        raise ValueError("median_rank: empty list")
    s = sorted(ranks)
    return max(1, s[(len(s) - 1) // 2])


def gen_mc_instance(m, n, r, s, sigma, seed, stream=0):
    """gen_mc_instance (P/include/dfc/simgen.hpp:45-59) with SeededRng(seed, stream)."""
    L0 = LowRankC()
    rows, cols, vals = i64ptr(), i64ptr(), C.POINTER(C.c_double)()
    _check(lib().dfcg_gen_mc_instance(i64(m), i64(n), i64(r), i64(s), C.c_double(sigma), u64(seed), u64(stream),
                                      C.byref(L0), C.byref(rows), C.byref(cols), C.byref(vals)))
    R = np.ctypeslib.as_array(rows, shape=(s,)).copy()
    Cc = np.ctypeslib.as_array(cols, shape=(s,)).copy()
    V = np.ctypeslib.as_array(vals, shape=(s,)).copy()
    for p in (rows, cols, vals):
        lib().dfcg_free(C.cast(p, C.c_void_p))
    return _lowrank_out(L0), Observed(m, n, R, Cc, V)


def _triplets_out(m, n, count, rows, cols, vals) -> Observed:
    N = int(count.value)
    if N:
        R = np.ctypeslib.as_array(rows, shape=(N,)).copy()
        Cc = np.ctypeslib.as_array(cols, shape=(N,)).copy()
        V = np.ctypeslib.as_array(vals, shape=(N,)).copy()
    else:
        R, Cc, V = np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0, np.float64)
    for p in (rows, cols, vals):
        lib().dfcg_free(C.cast(p, C.c_void_p))
    return Observed(int(m.value), int(n.value), R, Cc, V)


def parse_triplets(text, one_based=False) -> Observed:
    """load_triplets (P/include/dfc/matrix_io.hpp:125-170) on in-memory text: optional "% m n"
    header, one "i j v" line per observation; raises ParseError (.line), IndexError (outside the
    declared dims) or ValueError (no header and no data, duplicates) as the reference throws
    ParseError, std::out_of_range and std::invalid_argument."""
    raw = text.encode() if isinstance(text, str) else bytes(text)
    m, n, count = i64(), i64(), i64()
    rows, cols, vals = i64ptr(), i64ptr(), C.POINTER(C.c_double)()
    _check(lib().dfcg_load_triplets_text(C.c_char_p(raw), i64(len(raw)), C.c_int32(1 if one_based else 0),
                                         C.byref(m), C.byref(n), C.byref(count), C.byref(rows), C.byref(cols),
                                         C.byref(vals)))
    return _triplets_out(m, n, count, rows, cols, vals)


def load_triplets(path, one_based=False) -> Observed:
    """load_triplets on a file (memory-mapped, parsed and sorted on DFCG_IO_THREADS threads)."""
    m, n, count = i64(), i64(), i64()
    rows, cols, vals = i64ptr(), i64ptr(), C.POINTER(C.c_double)()
    _check(lib().dfcg_load_triplets_file(C.c_char_p(str(path).encode()), C.c_int32(1 if one_based else 0),
                                         C.byref(m), C.byref(n), C.byref(count), C.byref(rows), C.byref(cols),
                                         C.byref(vals)))
    return _triplets_out(m, n, count, rows, cols, vals)


def _obs_c(obs: Observed):
    from ._lib import ObsC

    R = np.ascontiguousarray(obs.rows, np.int64)
    Cc = np.ascontiguousarray(obs.cols, np.int64)
    V = np.ascontiguousarray(obs.vals, np.float64)
    return ObsC(obs.m, obs.n, len(V), _i(R), _i(Cc), _d(V)), (R, Cc, V)


def save_triplets(path, obs: Observed) -> None:
    """save_triplets (matrix_io.hpp:172-179): "% m n" then "row col %.17g" per entry."""
    oc, keep = _obs_c(obs)
    _check(lib().dfcg_save_triplets_file(C.c_char_p(str(path).encode()), C.byref(oc)))
    del keep


def format_triplets(obs: Observed) -> str:
    oc, keep = _obs_c(obs)
    text, n = C.c_void_p(), i64()
    _check(lib().dfcg_format_triplets(C.byref(oc), C.byref(text), C.byref(n)))
    out = C.string_at(text, n.value).decode()
    lib().dfcg_free(text)
    del keep
    return out


def gen_recsys_instance(m, n, r, density, seed, stream=0, cols=None, fsd=None, noise=0.8):
    """BASELINE c4 stand-in (dfcg_gen_recsys_instance): Zipf row/column popularity, values
    clip(round(3.6 + A B^T + N(0, noise^2)), 1, 5), A, B iid N(0, 0.3^2 / r); `cols` restricts the
    instance to a column subset (a D-step block; columns renumbered by subset position)."""
    fsd = 0.3 / np.sqrt(r) if fsd is None else fsd
    sub = np.asarray(cols if cols is not None else [], np.int64)
    cnt = i64()
    rows_p, cols_p, vals_p = i64ptr(), i64ptr(), C.POINTER(C.c_double)()
    _check(lib().dfcg_gen_recsys_instance(i64(m), i64(n), i64(r), C.c_double(density), C.c_double(fsd),
                                          C.c_double(noise), i64(len(sub)), _i(sub) if len(sub) else None,
                                          u64(seed), u64(stream), C.byref(cnt), C.byref(rows_p), C.byref(cols_p),
                                          C.byref(vals_p)))
    k = cnt.value
    R = np.ctypeslib.as_array(rows_p, shape=(max(k, 1),))[:k].copy()
    Cc = np.ctypeslib.as_array(cols_p, shape=(max(k, 1),))[:k].copy()
    V = np.ctypeslib.as_array(vals_p, shape=(max(k, 1),))[:k].copy()
    for p in (rows_p, cols_p, vals_p):
        lib().dfcg_free(C.cast(p, C.c_void_p))
    return Observed(m, len(sub) if len(sub) else n, R, Cc, V)


def gen_rmf_instance(m, n, r, s, sigma, seed, stream=0, lo=0.0, hi=1.0):
    """gen_rmf_instance (simgen.hpp:64-82); outliers U[lo, hi] (reference: U[0,1])."""
    L0 = LowRankC()
    S0 = SparseC()
    M = np.empty((m, n), np.float64, order="F")
    _check(lib().dfcg_gen_rmf_instance(i64(m), i64(n), i64(r), i64(s), C.c_double(sigma), u64(seed), u64(stream),
                                       C.c_double(lo), C.c_double(hi), C.byref(L0), C.byref(S0), _d(M)))
    cnt = S0.count
    rows = np.ctypeslib.as_array(S0.row, shape=(max(cnt, 1),))[:cnt].copy()
    cols = np.ctypeslib.as_array(S0.col, shape=(max(cnt, 1),))[:cnt].copy()
    vals = np.ctypeslib.as_array(S0.val, shape=(max(cnt, 1),))[:cnt].copy()
    lib().dfcg_sparse_free(C.byref(S0))
    return _lowrank_out(L0), (rows, cols, vals), M


# ------------------------------------------------------------------ kernel accounting
PROF_OPS = ("gemm", "sddmm", "spmm", "cholesky", "qr_fallback", "jacobi", "elementwise", "reduce", "other",
            "gemm_small")


def prof_enable(on: bool = True):
    """Start (and clear) / stop CUDA-event accounting of every library op (bench only)."""
    lib().dfcg_prof_enable(C.c_int(1 if on else 0))


def prof_collect() -> dict:
    """{op: dict(launches, ms, flops, bytes)} since the last prof_enable(True)."""
    n = len(PROF_OPS)
    launches = np.zeros(n, np.int64)
    ms, fl, by = np.zeros(n), np.zeros(n), np.zeros(n)
    rc = lib().dfcg_prof_collect(_i(launches), _d(ms), _d(fl), _d(by))
    if rc < 0:
        _check(rc)
    return {op: dict(launches=int(launches[i]), ms=float(ms[i]), flops=float(fl[i]), bytes=float(by[i]))
            for i, op in enumerate(PROF_OPS)}


def work_counters() -> dict:
    """{op: dict(launches, flops, bytes)}: cumulative always-on counters (no events)."""
    n = len(PROF_OPS)
    launches = np.zeros(n, np.int64)
    fl, by = np.zeros(n), np.zeros(n)
    _check(min(0, lib().dfcg_work_counters(_i(launches), _d(fl), _d(by))))
    return {op: dict(launches=int(launches[i]), flops=float(fl[i]), bytes=float(by[i]))
            for i, op in enumerate(PROF_OPS)}


def launch_count() -> int:
    """Total kernels launched by libdfcg in this process."""
    lib().dfcg_launch_count.restype = i64
    return int(lib().dfcg_launch_count())
