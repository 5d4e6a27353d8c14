"""Warm-started CholeskyQR over a whole c2 block solve (run with DFCG_TRACE_CHOLQR=1): every
factorisation's smallest scaled pivot and the accumulated pair's max |R Rinv - I| go to stderr;
this prints the solve's iteration count, rank and time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P  # noqa: E402

L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
blk = P.extract_columns(obs, P.partition_columns(1, 0xDFC0000000000001, 10000, 8)[0])
del obs
sv = P.McSolver(blk)
t0 = time.time()
done, tr = sv.step(500, trace=True)
print(f"{done} iterations, final rank {tr[-1]['rank']}, rel {tr[-1]['rel']:.3e}, {time.time() - t0:.1f} s", flush=True)
sv.close()
