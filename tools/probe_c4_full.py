"""BASELINE c4 at its full size on one GPU: the recommender-shaped stand-in (no reference generator
exists) — 17770 x 480189, ~1.17% observed (~1e8 cells, Zipf(1) row and column
popularity), r = 30, ratings clip(round(3.6 + A B^T + N(0, 0.8^2)), 1, 5) — generated whole
(gen_recsys_instance), then the whole DFC-Proj pipeline with t = 64 column blocks through the C ABI
(dfc_run: D step, the 64 blocks solved concurrently on one GPU, column_project).

Solver: the reference's noisy-MC block floor (P/tests/acceptance.cpp:127-130),
mu_floor = sigma sqrt(rho) (sqrt(m) + sqrt(n / t)) with sigma = 0.8; under the default floor the c4
blocks climb to rank ~1900 within 15 iterations (r01 probe, profiles/r01_c4_standin_blocks.txt) and a
500-iteration solve of 64 blocks would take hours on one GPU. Prints the phases, per-block
iteration / rank spread, nnz skew and the RMSE on 2e5 held-in cells against the noiseless rating."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1107_0789_b200 as P  # noqa: E402

t_blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 64
workers = int(sys.argv[2]) if len(sys.argv) > 2 else 16
m, n, r, dens, sigma = 17770, 480189, 30, 0.0117, 0.8
t0 = time.time()
obs = P.gen_recsys_instance(m, n, r, dens, 1)
gen_s = time.time() - t0
print(f"gen {gen_s:.1f}s nnz {obs.count} ({obs.count / (m * n):.4%})", flush=True)
rho = obs.count / (m * n)
floor = sigma * math.sqrt(rho) * (math.sqrt(m) + math.sqrt(n / t_blocks))
t0 = time.time()
est, info = P.dfc_run(obs, "proj", t=t_blocks, seed=1, workers=workers, solver_cfg=P.ApgConfig(mu_floor=floor))
wall = time.time() - t0
its = [x.iterations for x in info["subproblems"]]
ranks = [x.rank for x in info["subproblems"]]
rng = np.random.default_rng(0)
sel = rng.integers(0, obs.count, 200_000)
pred = np.einsum("ij,ij->i", est.left[obs.rows[sel]], est.right[obs.cols[sel]])
rmse_obs = float(np.sqrt(np.mean((pred - obs.vals[sel]) ** 2)))
groups = P.partition_columns(1, 0xDFC0000000000001, n, t_blocks)
col_nnz = np.bincount(obs.cols, minlength=n)
blk_nnz = [int(col_nnz[g].sum()) for g in groups]
row = dict(config=f"c4 stand-in {m}x{n} r={r} density {rho:.4%} DFC-Proj t={t_blocks}", gen_s=round(gen_s, 1),
           mu_floor=round(floor, 3), solve_s=round(wall, 2), divide_ms=round(info["divide_ms"], 1),
           factor_ms=round(info["factor_ms"], 1), combine_ms=round(info["combine_ms"], 1),
           block_iterations=sum(its), iterations_min_max=[min(its), max(its)],
           block_it_per_s=round(sum(its) / (info["factor_ms"] * 1e-3), 1), ranks_min_max=[min(ranks), max(ranks)],
           rank=est.rank, block_nnz_min_max=[min(blk_nnz), max(blk_nnz)], rmse_on_observed=round(rmse_obs, 4),
           workers=workers)
print(json.dumps(row), flush=True)
