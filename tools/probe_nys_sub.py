"""Per-op cost of the two DFC-Nys subproblems at c2 (C-hat 10000 x 1250, R-hat 1250 x 10000), each
run alone: iterations 1..N, then one profiled iteration."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1107_0789_b200 as P
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
cols = np.sort(P.sample_without_replacement(1, 0xDFC0000000000002, 10000, 1250))
rows = np.sort(P.sample_without_replacement(1, 0xDFC0000000000003, 10000, 1250))
for name, sub in (("C-hat", P.extract_columns(obs, cols)), ("R-hat", P.extract_rows(obs, rows))):
    s = P.McSolver(sub, P.ApgConfig())
    t0 = time.time()
    done, tr = s.step(iters, trace=True)
    dt = time.time() - t0
    print(f"{name} {sub.m}x{sub.n} nnz {sub.count}: {done} its {dt:.2f}s, last ranks {[t['rank'] for t in tr[-5:]]} "
          f"ms {[round(t['ms'], 1) for t in tr[-5:]]}", flush=True)
    P.prof_enable(True)
    s.step(1)
    prof = P.prof_collect()
    P.prof_enable(False)
    tot = sum(v['ms'] for v in prof.values())
    for op, v in sorted(prof.items(), key=lambda kv: -kv[1]['ms']):
        if v['launches']:
            print(f"   {op:12s} launches {v['launches']:5d} ms {v['ms']:7.2f} ({100*v['ms']/tot:4.1f}%) "
                  f"{v['flops']/(v['ms']*1e-3)/1e12:6.2f} TF/s", flush=True)
    s.close()
