"""DFC-Nys row subproblem at c2 (1250 x 10000) run twice in one process: the second run reads a
fully generated normal-stream cache, isolating the generator's share of the iteration time."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1107_0789_b200 as P
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
rows = np.sort(P.sample_without_replacement(1, 0xDFC0000000000003, 10000, 1250))
sub = P.extract_rows(obs, rows)
for run in range(2):
    s = P.McSolver(sub, P.ApgConfig())
    t0 = time.time()
    done, tr = s.step(iters, trace=True)
    print(f"run {run}: {done} its {time.time() - t0:.2f}s; its {iters-10}..{iters}: ms " +
          " ".join(f"{t['ms']:.0f}/c{t['svd_calls']}" for t in tr[-10:]), flush=True)
    s.close()
