"""The reference's experiment harness (run_experiment / write_csv / results_to_json,
P/include/dfc/bench.hpp:24-386) on the GPU path: same methods, seeds, instance streams, timing
columns, RMSE definition, per-method mean/std summary rows and the same CSV / JSON schema, so
result files are drop-in comparable with the reference's `method,seed,rmse,ms_*,rank` output.

Methods (bench.hpp:24-38): base (one apg_mc / apg_rmf on the whole matrix), part (the F step
only: block estimates placed back at their columns, bench.hpp:106-127), proj / proj-ens, rp /
rp-ens, nys / nys-ens (dfc_run)."""
from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L
from . import host as H

METHODS = ("base", "part", "proj", "proj-ens", "rp", "rp-ens", "nys", "nys-ens")
PARTITION_STREAM = 0xDFC0000000000001  # streams::partition (P/include/dfc/dfc.hpp)


@dataclass
class ExperimentSpec:
    """ExperimentSpec (bench.hpp:53-75) for generated instances."""
    task: str = "mc"
    m: int = 0
    n: int = 0
    r: int = 0
    s: int = 0
    sigma: float = 0.0
    methods: List[str] = field(default_factory=lambda: ["proj"])
    seeds: List[int] = field(default_factory=lambda: [1])
    t: int = 4
    l_frac: float = 0.1
    d_frac: float = 0.1
    p: int = 5
    q: int = 2
    workers: int = 1
    solver_cfg: Optional[L.ApgConfig] = None
    lam: float = 0.0
    device: int = 0


@dataclass
class ResultRow:
    method: str
    seed: int
    rmse: float = 0.0
    ms_divide: float = 0.0
    ms_factor: float = 0.0
    ms_combine: float = 0.0
    ms_total: float = 0.0
    rank: int = 0
    config_echo: str = ""


def _validate(spec: ExperimentSpec):  # detail::validate_spec, bench.hpp:129-140
    if not spec.seeds:
        raise ValueError("ExperimentSpec: seeds must be nonempty")
    if not spec.methods:
        raise ValueError("ExperimentSpec: methods must be nonempty")
    if not (0 < spec.l_frac <= 1) or not (0 < spec.d_frac <= 1):
        raise ValueError("ExperimentSpec: sampling fractions must be in (0,1]")
    if spec.t < 1:
        raise ValueError("ExperimentSpec: t must be >= 1")
    if spec.workers < 1:
        raise ValueError("ExperimentSpec: workers must be >= 1")
    if spec.m < 1 or spec.n < 1 or spec.r < 1 or spec.s < 1:
        raise ValueError("ExperimentSpec: generated instances need m, n, r, s")
    for mth in spec.methods:
        if mth not in METHODS:
            raise ValueError(f"unknown method '{mth}'")


def config_echo(spec: ExperimentSpec) -> str:  # detail::config_echo, bench.hpp:142-153
    return (f"task={spec.task};m={spec.m};n={spec.n};r={spec.r};s={spec.s};sigma={spec.sigma:g}"
            f";t={spec.t};l_frac={spec.l_frac:g};d_frac={spec.d_frac:g};p={spec.p};q={spec.q}"
            f";workers={spec.workers}")


def factored_rmse(truth, est, m, n) -> float:
    """rmse (bench.hpp:80-85): factored_diff_norm / sqrt(m n), with the reference's cancellation
    formula ||a||^2 - 2 <a, b> + ||b||^2 clamped at 0 (solvers.hpp:179-193)."""
    def inner(al, ar, bl, br):
        if al.shape[1] == 0 or bl.shape[1] == 0:
            return 0.0
        return float(np.sum((al.T @ bl) * (ar.T @ br)))
    d2 = (inner(truth.left, truth.right, truth.left, truth.right)
          - 2.0 * inner(truth.left, truth.right, est.left, est.right)
          + inner(est.left, est.right, est.left, est.right))
    return math.sqrt(max(0.0, d2)) / math.sqrt(float(m) * float(n))


def assemble_blocks(ests, groups, m, n, device=0):
    """detail::assemble_blocks (bench.hpp:106-127): block estimates at their original columns,
    compacted by svd_of_product when the stacked rank exceeds min(m, n)."""
    total_k = sum(e.rank for e in ests)
    if total_k == 0:
        return L.Estimate(np.zeros((m, 0)), np.zeros((n, 0)))
    left = np.zeros((m, total_k))
    right = np.zeros((n, total_k))
    at = 0
    for e, idx in zip(ests, groups):
        k = e.rank
        if k == 0:
            continue
        left[:, at:at + k] = e.left
        right[np.asarray(idx), at:at + k] = e.right
        at += k
    if total_k > min(m, n):
        return L.svd_of_product(left, right, device=device)[0]
    return L.Estimate(left, right)


def run_experiment(spec: ExperimentSpec) -> List[ResultRow]:
    """run_experiment (bench.hpp:158-336) with the F and C steps on the GPU."""
    _validate(spec)
    echo = config_echo(spec)
    cfg = spec.solver_cfg or L.ApgConfig()
    rows: List[ResultRow] = []
    for method in spec.methods:
        for seed in spec.seeds:
            # instance on SeededRng(seed, 0) (orchestrator streams are disjoint)
            if spec.task == "mc":
                truth, obs = H.gen_mc_instance(spec.m, spec.n, spec.r, spec.s, spec.sigma, seed)
                M = None
            else:
                truth, _S0, M = H.gen_rmf_instance(spec.m, spec.n, spec.r, spec.s, spec.sigma, seed)
                ii, jj = np.meshgrid(np.arange(spec.m), np.arange(spec.n), indexing="ij")
                obs = L.Observed(spec.m, spec.n, ii.T.ravel().astype(np.int64), jj.T.ravel().astype(np.int64),
                                 np.asarray(M, order="F").T.ravel().copy())
            row = ResultRow(method, int(seed), config_echo=echo)
            if method == "base":
                if spec.task == "mc":
                    est, rep = L.apg_mc(obs, cfg, device=spec.device)
                else:
                    lam = spec.lam if spec.lam > 0 else 1.0 / math.sqrt(max(spec.m, spec.n))
                    est, _S, rep = L.apg_rmf(np.asfortranarray(M), lam, cfg, device=spec.device)
                row.ms_factor = row.ms_total = rep.wall_ms
                row.rank = rep.rank
            elif method == "part":
                t0 = time.perf_counter()
                groups = H.partition_columns(seed, PARTITION_STREAM, obs.n, min(spec.t, obs.n))
                blocks = [H.extract_columns(obs, g) for g in groups]
                t1 = time.perf_counter()
                if spec.task == "mc":
                    ests = [L.apg_mc(b, cfg, device=spec.device)[0] for b in blocks]
                else:
                    ests = []
                    for g in groups:
                        Mb = np.asfortranarray(M[:, g])
                        lam = spec.lam if spec.lam > 0 else 1.0 / math.sqrt(max(Mb.shape))
                        ests.append(L.apg_rmf(Mb, lam, cfg, device=spec.device)[0])
                t2 = time.perf_counter()
                est = assemble_blocks(ests, groups, obs.m, obs.n, spec.device)
                t3 = time.perf_counter()
                row.ms_divide, row.ms_factor, row.ms_combine = 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2)
                row.ms_total = 1e3 * (t3 - t0)
                row.rank = est.rank
            else:
                variant = method.split("-")[0]
                est, info = L.dfc_run(obs, variant=variant, ensemble=method.endswith("-ens"),
                                      t=min(spec.t, obs.n),
                                      l=max(1, int(round(spec.l_frac * obs.n))),
                                      d=max(1, int(round(spec.d_frac * obs.m))),
                                      rp_p=spec.p, rp_q=spec.q, seed=seed, solver_cfg=cfg, task=spec.task,
                                      lam=spec.lam, workers=spec.workers, device=spec.device)
                row.ms_divide, row.ms_factor = info["divide_ms"], info["factor_ms"]
                row.ms_combine, row.ms_total = info["combine_ms"], info["total_ms"]
                row.rank = est.rank
            row.rmse = factored_rmse(truth, est, obs.m, obs.n)
            rows.append(row)
    rows.sort(key=lambda r: (r.method, r.seed))
    summary = []
    for method in spec.methods:  # mean / std rows per method (bench.hpp:292-334)
        group = [r for r in rows if r.method == method]
        if not group:
            continue
        cnt = len(group)
        mean = ResultRow(method + "_mean", cnt, config_echo=echo)
        std = ResultRow(method + "_std", cnt, config_echo=echo)
        for f in ("rmse", "ms_divide", "ms_factor", "ms_combine", "ms_total"):
            vals = [getattr(r, f) for r in group]
            mu = sum(vals) / cnt
            setattr(mean, f, mu)
            setattr(std, f, math.sqrt(sum((v - mu) ** 2 for v in vals) / (cnt - 1)) if cnt > 1 else 0.0)
        mean.rank = int(round(sum(r.rank for r in group) / cnt))
        summary += [mean, std]
    summary.sort(key=lambda r: r.method)
    return rows + summary


def write_csv(out, rows: List[ResultRow]):
    """write_csv (bench.hpp:339-351): header and number formats of the reference."""
    out.write("method,seed,rmse,ms_divide,ms_factor,ms_combine,ms_total,rank\n")
    for r in rows:
        out.write(f"{r.method},{r.seed},{r.rmse:.12g},{r.ms_divide:.6g},{r.ms_factor:.6g},{r.ms_combine:.6g},"
                  f"{r.ms_total:.6g},{r.rank}\n")


def results_to_json(spec: ExperimentSpec, rows: List[ResultRow]) -> str:
    """results_to_json (bench.hpp:353-384)."""
    cfg = dict(task=spec.task, m=spec.m, n=spec.n, r=spec.r, s=spec.s, sigma=spec.sigma, input="",
               methods=list(spec.methods), t=spec.t, l_frac=spec.l_frac, d_frac=spec.d_frac, p=spec.p,
               q=spec.q, workers=spec.workers, seeds=list(spec.seeds))
    jrows = [dict(method=r.method, seed=r.seed, rmse=r.rmse, ms_divide=r.ms_divide, ms_factor=r.ms_factor,
                  ms_combine=r.ms_combine, ms_total=r.ms_total, rank=r.rank, config=r.config_echo) for r in rows]
    return json.dumps(dict(config=cfg, rows=jrows))
