"""Per-block APG trajectories of the c2 workload (rank, k, SVT calls, ms per iteration)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 60
L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
groups = P.partition_columns(1, 0xDFC0000000000001, 10000, 8)
for g in range(int(sys.argv[2]) if len(sys.argv) > 2 else 8):
    blk = P.extract_columns(obs, groups[g])
    est, rep = P.apg_mc(blk, P.ApgConfig(max_iters=iters))
    calls = [t['svd_calls'] for t in rep.trace]
    ms = [t['ms'] for t in rep.trace]
    ks = [t['k_final'] for t in rep.trace]
    print(f"block {g}: multi-call iterations {[i + 1 for i, c in enumerate(calls) if c > 1]}")
    print("  ms  " + " ".join(f"{x:.0f}" for x in ms))
    print("  k   " + " ".join(str(x) for x in ks))
