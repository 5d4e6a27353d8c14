"""Generate the BASELINE-scale oracle fixtures (TEST INFRASTRUCTURE: runs the CPU oracle only).

The oracle (oracle/, the restated reference) is too slow to run inside a GPU test at the
BASELINE block sizes, so its trajectories are recorded here once and committed as small
fixtures; tests/test_gpu_baseline_scale.py runs the CUDA path on the same seed-generated
inputs and compares.

  c2_window: BASELINE c2 (gen_mc_instance(1e4, 1e4, 10, 1e7, 0.1), seed 1, DFC-Proj t = 8
             partition, P/include/dfc/dfc.hpp:166-200), block 0 (10000 x 1250) under the
             default ApgConfig, the first ITERS APG iterations (apg_mc,
             P/include/dfc/solvers.hpp:241-327) — through the rank ~700 window bench.py times.
  c3_block:  BASELINE c3 (gen_rmf_instance variant: outliers U[-10, 10], sigma 0.01, 10%
             outliers, seed 1), block 0 (10000 x 1250) solved to convergence by apg_rmf
             (P/include/dfc/solvers.hpp:332-414) with lambda = 1/sqrt(max(m, w))
             (P/include/dfc/dfc.hpp:74).

Each fixture stores the per-iteration trace (rank, k of the last partial SVD, SVD calls,
rel, mu, sum of singular values), the final report, and sketches of the final estimates:
Lᵀ·X (w x 16) for X = SeededRng(PROBE_SEED, 0) normals (m x 16, column-major), plus the
Frobenius norms. ||(L_gpu - L_oracle)ᵀ X||_F / ||L_oracleᵀ X||_F estimates the relative
Frobenius error (E||EᵀX||² = 16 ||E||_F²) without committing the m x k factors.

  base_full: the reference's "Base" method (apg_mc on the WHOLE matrix, P/include/dfc/bench.hpp:
             211-217) at BASELINE c2 (10000 x 10000, 1e7 observations), default ApgConfig, the
             first ITERS iterations (ranks 1 .. ~1450; the next iteration jumps to k ~ 5800,
             beyond what the oracle finishes in minutes).

usage: python tests/golden/make_fixtures.py c2_window|c3_block|base_full [--iters N] [--threads T]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402

PARTITION_STREAM = 0xDFC0000000000001
PROBE_SEED = 0x5EED
NPROBE = 16


def probes(m: int) -> np.ndarray:
    return O.rng_normal(PROBE_SEED, 0, m * NPROBE).reshape(NPROBE, m).T  # m x 16, column-major draw order


def c2_block0():
    L0, obs = O.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
    groups = O.partition_columns(1, PARTITION_STREAM, 10000, 8)
    return O.extract_columns(obs, groups[0])


def c3_block0():
    L0, S0, M = O.gen_rmf_instance(10000, 10000, 10, 10_000_000, 0.01, 1, lo=-10.0, hi=10.0)
    groups = O.partition_columns(1, PARTITION_STREAM, 10000, 8)
    return np.asfortranarray(M[:, groups[0]])


def sketch(left: np.ndarray, right: np.ndarray, X: np.ndarray) -> np.ndarray:
    return right @ (left.T @ X)  # (L^T X), w x 16


def fro_lowrank(left, right) -> float:
    return float(np.sqrt(max(np.sum((left.T @ left) * (right.T @ right)), 0.0)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["c2_window", "c3_block", "base_full"])
    ap.add_argument("--iters", type=int, default=45)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    O.lib().orc_set_blas_threads(args.threads)
    t0 = time.time()
    if args.which in ("c2_window", "base_full"):
        if args.which == "c2_window":
            blk = c2_block0()
        else:
            L0, blk = O.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
        run = O.McRun(blk)
        trace = []
        for i in range(args.iters):
            trace += run.step(1)
            print(f"[{time.time() - t0:7.1f}s] it {trace[-1]['it']} rank {trace[-1]['rank']} "
                  f"k {trace[-1]['k_final']} calls {trace[-1]['svd_calls']}", flush=True)
        est, rep = run.finish()
        X = probes(blk.m)
        out = dict(which=args.which, m=blk.m, n=blk.n, nnz=blk.count, iters=args.iters, trace=trace,
                   report=dict(iterations=rep.iterations, rank=rep.rank, objective=rep.objective,
                               residual=rep.residual),
                   fro_L=fro_lowrank(est.left, est.right),
                   sigma=np.linalg.norm(est.right, axis=0).tolist())
        np.save(os.path.join(HERE, f"{args.which}_LtX.npy"), sketch(est.left, est.right, X))
    else:
        M = c3_block0()
        lam = 1.0 / np.sqrt(max(M.shape))
        est, S, rep = O.apg_rmf(M, lam)
        X = probes(M.shape[0])
        rows, cols, vals = S
        StX = np.zeros((M.shape[1], NPROBE))
        np.add.at(StX, cols, vals[:, None] * X[rows])
        out = dict(which="c3_block", m=M.shape[0], n=M.shape[1], lam=lam, trace=rep.trace,
                   report=dict(iterations=rep.iterations, rank=rep.rank, objective=rep.objective,
                               residual=rep.residual),
                   fro_L=fro_lowrank(est.left, est.right), fro_S=float(np.linalg.norm(vals)),
                   nnz_S=int(len(vals)), sum_S=float(np.sum(vals)),
                   sigma=np.linalg.norm(est.right, axis=0).tolist())
        np.save(os.path.join(HERE, "c3_block_LtX.npy"), sketch(est.left, est.right, X))
        np.save(os.path.join(HERE, "c3_block_StX.npy"), StX)
    out["oracle_seconds"] = time.time() - t0
    out["oracle_threads"] = args.threads
    out["generator"] = "tests/golden/make_fixtures.py"
    with open(os.path.join(HERE, f"{args.which}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()
