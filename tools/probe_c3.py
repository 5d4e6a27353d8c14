"""Time one BASELINE c3 RMF block (10000 x 1250 dense, 10% outliers U[-10,10], noise 0.01)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1107_0789_b200 as P
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
m, w = 10000, 1250
t0 = time.time()
L0, S0, M = P.gen_rmf_instance(m, w, 10, m * w // 10, 0.01, 1, lo=-10.0, hi=10.0)
print(f"gen {time.time()-t0:.1f}s", flush=True)
lam = 1.0 / np.sqrt(max(m, w))
t0 = time.time()
est, S, rep = P.apg_rmf(M, lam, P.ApgConfig(max_iters=iters))
print(f"apg_rmf {rep.iterations} its: {time.time()-t0:.2f}s rank={rep.rank} nnzS={len(S[2])}", flush=True)
for t in rep.trace[-8:]:
    print(f"it {t['it']:4d} rank {t['rank']:5d} k {t['k_final']:5d} calls {t['svd_calls']} rel {t['rel']:.3e} ms {t['ms']:.1f}")
P.prof_enable(True)
est, S, rep = P.apg_rmf(M, lam, P.ApgConfig(max_iters=5))
prof = P.prof_collect()
P.prof_enable(False)
tot = sum(v['ms'] for v in prof.values())
for op, v in sorted(prof.items(), key=lambda kv: -kv[1]['ms']):
    if v['launches'] == 0: continue
    print(f"{op:12s} launches {v['launches']:6d} ms {v['ms']:8.1f} ({100*v['ms']/tot:5.1f}%) "
          f"{v['flops']/(v['ms']*1e-3)/1e12 if v['ms'] else 0:6.2f} TFLOP/s {v['bytes']/(v['ms']*1e-3)/1e9 if v['ms'] else 0:8.1f} GB/s")
