"""Time one BASELINE c2 block (10000 x 1250, default ApgConfig) on the GPU with a trace."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1107_0789_b200 as P
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
t0 = time.time()
L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
groups = P.partition_columns(1, 0xDFC0000000000001, 10000, 8)
blk = P.extract_columns(obs, groups[0])
print(f"gen+extract {time.time()-t0:.1f}s nnz={blk.count}", flush=True)
t0 = time.time()
est, rep = P.apg_mc(blk, P.ApgConfig(max_iters=iters))
print(f"apg_mc {iters} its: {time.time()-t0:.2f}s wall_ms={rep.wall_ms:.0f} rank={rep.rank}", flush=True)
for t in rep.trace:
    print(f"it {t['it']:4d} rank {t['rank']:5d} k {t['k_final']:5d} calls {t['svd_calls']} rel {t['rel']:.3e} ms {t['ms']:.1f}")

# profile a second window of iterations with per-op accounting
P.prof_enable(True)
t0 = time.time()
est, rep = P.apg_mc(blk, P.ApgConfig(max_iters=iters))
wall = time.time() - t0
prof = P.prof_collect()
P.prof_enable(False)
print(f"profiled run wall {wall:.2f}s")
tot = sum(v['ms'] for v in prof.values())
for op, v in sorted(prof.items(), key=lambda kv: -kv[1]['ms']):
    if v['launches'] == 0: continue
    tf = v['flops'] / (v['ms'] * 1e-3) / 1e12 if v['ms'] > 0 else 0
    gb = v['bytes'] / (v['ms'] * 1e-3) / 1e9 if v['ms'] > 0 else 0
    print(f"{op:12s} launches {v['launches']:7d} ms {v['ms']:9.1f} ({100*v['ms']/tot:5.1f}%) {tf:6.2f} TFLOP/s {gb:8.1f} GB/s")
print("launch count", P.launch_count())
