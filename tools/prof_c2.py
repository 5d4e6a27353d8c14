"""Short c2-block run for ncu / SVD tracing (iterations 1..N of block 0)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 12
L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
groups = P.partition_columns(1, 0xDFC0000000000001, 10000, 8)
blk = P.extract_columns(obs, groups[0])
est, rep = P.apg_mc(blk, P.ApgConfig(max_iters=iters))
print("iters", rep.iterations, "rank", rep.rank, "wall_ms", rep.wall_ms)
