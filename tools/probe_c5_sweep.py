"""BASELINE c5 scaling sweep on one GPU: DFC-Proj-Ens on the full 40000 x 40000 instance (reference
generator gen_mc_instance: r = 20, 5% observed = 8e7 cells, sigma 0.1, seed 1), t in {8, 16, 32, 64}
column blocks, the combine projecting every block onto the first 4 blocks' column spaces (BASELINE
"ensemble of 4", DfcConfig ensemble_anchors = 4) and recompressing to the median block rank.

Solver: the reference's block configuration of its noisy-MC acceptance grid
(P/tests/acceptance.cpp:127-130): mu_floor = sigma sqrt(rho) (sqrt(m) + sqrt(n / t)). Under the
default floor (1e-4 mu_init) the c5 blocks climb to rank ~3400 within 7 iterations (r01 probe) and
a 500-iteration solve of 64 such blocks is hours per t; the acceptance floor converges in ~100
iterations at rank ~20, where the per-iteration work is the SDDMM / SpMM over 1e7 / t observations.

Every t: the whole dfc_run through the C ABI (host triplets in, host factors out; D step, F step
with t blocks concurrently on the GPU, combine), its phases, block-iterations/s of the F step, the
final rank, and the RMSE of the estimate against L0 on 2e5 random cells."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1107_0789_b200 as P  # noqa: E402

ts = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [8, 16, 32, 64]
anchors = int(sys.argv[2]) if len(sys.argv) > 2 else 4
m = n = 40000
r, s, sigma = 20, 80_000_000, 0.1
t0 = time.time()
L0, obs = P.gen_mc_instance(m, n, r, s, sigma, 1)
print(f"gen {time.time() - t0:.1f}s nnz {obs.count}", flush=True)
rng = np.random.default_rng(0)
I, J = rng.integers(0, m, 200_000), rng.integers(0, n, 200_000)
truth = np.einsum("ij,ij->i", L0.left[I], L0.right[J])
rho = s / (m * n)
rows = []
for t in ts:
    floor = sigma * math.sqrt(rho) * (math.sqrt(m) + math.sqrt(n / t))
    # Continuation start: the reference's mu_init = 0.99 ||P_Omega M_b||_2 (solvers.hpp:259) sits
    # within the randomized range finder's sigma_1 error on these narrow, sparse blocks, so the
    # first SVT returns rank 0 and apg_mc stops after one iteration with a zero estimate (the
    # reference does the same, r01 parity probe). The sweep starts continuation at 0.9 sigma_1 of
    # block 0 instead (ApgConfig::mu_init, one value for every block).
    g0 = P.partition_columns(1, 0xDFC0000000000001, n, t)[0]
    sv = P.McSolver(P.extract_columns(obs, g0), P.ApgConfig(max_iters=1))
    _, tr = sv.step(1, trace=True)
    sv.close()
    mu_init = tr[0]["mu"] * 0.90 / 0.99
    cfg = P.ApgConfig(mu_floor=floor, mu_init=mu_init)
    t1 = time.time()
    est, info = P.dfc_run(obs, "proj", ensemble=True, ensemble_anchors=anchors, t=t, seed=1, workers=min(t, 16),
                          solver_cfg=cfg)
    wall = time.time() - t1
    its = [x.iterations for x in info["subproblems"]]
    pred = np.einsum("ij,ij->i", est.left[I], est.right[J])
    rmse = float(np.sqrt(np.mean((pred - truth) ** 2)))
    row = dict(t=t, anchors=anchors, mu_floor=round(floor, 4), mu_init=round(mu_init, 3), solve_s=round(wall, 2),
               divide_ms=round(info["divide_ms"], 1), factor_ms=round(info["factor_ms"], 1),
               combine_ms=round(info["combine_ms"], 1), block_iterations=sum(its),
               iterations_min_max=[min(its), max(its)],
               block_it_per_s=round(sum(its) / (info["factor_ms"] * 1e-3), 1), rank=est.rank,
               block_ranks_min_max=[min(x.rank for x in info["subproblems"]),
                                    max(x.rank for x in info["subproblems"])], rmse=round(rmse, 5))
    rows.append(row)
    print(json.dumps(row), flush=True)
print(json.dumps(dict(config="c5 DFC-Proj-Ens 40000x40000 r=20 8e7 obs sigma=0.1 seed 1, ensemble of "
                             f"{anchors}, acceptance-style block floor", rows=rows)))
