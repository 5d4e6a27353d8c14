"""Time DFC-Nys at BASELINE c2 (10000 x 10000, r=10, 10% observed, l = d = 1250) through dfc_run."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1107_0789_b200 as P
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 500
t0 = time.time()
L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
print(f"gen {time.time()-t0:.1f}s", flush=True)
for variant, kw in (("nys", dict(l=1250, d=1250)), ("proj", dict(t=8))):
    t0 = time.time()
    est, info = P.dfc_run(obs, variant=variant, seed=1, solver_cfg=P.ApgConfig(max_iters=iters), workers=8, **kw)
    wall = time.time() - t0
    its = sum(s.iterations for s in info["subproblems"])
    print(f"{variant}: wall {wall:.2f}s factor {info['factor_ms']/1e3:.2f}s combine {info['combine_ms']:.1f}ms "
          f"rank {est.rank} subproblem iterations {[s.iterations for s in info['subproblems']]} "
          f"ranks {[s.rank for s in info['subproblems']]} -> {its / (info['factor_ms'] * 1e-3):.1f} it/s", flush=True)
