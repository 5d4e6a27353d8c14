"""Run the c2 block under the acceptance floor for N iterations (for ncu: DFCG_PROFILE_ITER)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 70
L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
groups = P.partition_columns(1, 0xDFC0000000000001, 10000, 8)
blk = P.extract_columns(obs, groups[0])
floor = 0.1 * math.sqrt(0.1) * (math.sqrt(10000) + math.sqrt(1250))
est, rep = P.apg_mc(blk, P.ApgConfig(mu_floor=floor, max_iters=iters))
print("iters", rep.iterations, "rank", rep.rank)
