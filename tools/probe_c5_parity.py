"""BASELINE c5 full instance (40000 x 40000, r = 20, 8e7 cells): blocks 1 and 0 of the t = 8
partition, the first three APG iterations on the GPU and in the CPU oracle (rank, k, calls, mu,
sum of singular values) -- parity at the c5 block size."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1107_0789_b200 as P
import oracle as O
m = n = 40000
L0, obs = P.gen_mc_instance(m, n, 20, 80_000_000, 0.1, 1)
groups = P.partition_columns(1, 0xDFC0000000000001, n, 8)
for g in (1, 0):
    blk = P.extract_columns(obs, groups[g])
    est, rep = P.apg_mc(blk, P.ApgConfig(max_iters=3))
    print("gpu block", g, [(t["rank"], t["k_final"], t["svd_calls"], round(t["mu"], 6), t["sigma_sum"]) for t in rep.trace], flush=True)
    t0 = time.time()
    eo, ro = O.apg_mc(O.Observed(blk.m, blk.n, blk.rows, blk.cols, blk.vals), O.apg_cfg(max_iters=3))
    print("oracle block", g, [(t["rank"], t["k_final"], t["svd_calls"], round(t["mu"], 6), t["sigma_sum"]) for t in ro.trace], f"{time.time()-t0:.1f}s", flush=True)
