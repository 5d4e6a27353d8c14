"""Base APG (the reference's "Base" method, P/include/dfc/bench.hpp:211-217: apg_mc on the WHOLE
matrix) at BASELINE c2: 10000 x 10000, r = 10, 1e7 observations, default ApgConfig. Runs the
resumable solver for up to --iters iterations or --budget seconds and prints the per-iteration
trace (rank, k, SVD calls, host ms) — sizing for bench.py's base_apg line."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=60)
ap.add_argument("--budget", type=float, default=240.0)
ap.add_argument("--prof", action="store_true")
a = ap.parse_args()
t0 = time.time()
L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
print(f"gen {time.time() - t0:.1f}s nnz={obs.count}", flush=True)
t0 = time.time()
sv = P.McSolver(obs)
print(f"setup {time.time() - t0:.2f}s", flush=True)
t0 = time.time()
done = 0
while done < a.iters and time.time() - t0 < a.budget:
    if a.prof:
        P.prof_enable(True)
    n, tr = sv.step(1, trace=True)
    if not n:
        break
    done += n
    t = tr[-1]
    line = (f"it {t['it']:4d} rank {t['rank']:5d} k {t['k_final']:5d} calls {t['svd_calls']} rel {t['rel']:.3e} "
            f"ms {t['ms']:9.1f} t {time.time() - t0:7.1f}s")
    if a.prof:
        prof = P.prof_collect()
        P.prof_enable(False)
        line += " | " + " ".join(f"{k}:{v['ms']:.0f}ms/{v['launches']}" for k, v in
                                 sorted(prof.items(), key=lambda kv: -kv[1]['ms']) if v['launches'])
    print(line, flush=True)
est, rep = sv.finish()
sv.close()
print(f"{done} iterations in {time.time() - t0:.1f}s: {done / (time.time() - t0):.3f} it/s, rank {rep.rank}")
