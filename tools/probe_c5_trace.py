"""Per-iteration trace of one c5-shaped block (40000 x 5000, N = 1e7, r = 20, sigma 0.1) under the
sweep's solver configuration (acceptance-style floor, continuation from 0.9 sigma_1): iteration,
rank, k, SVD calls, host ms — where the 186 iterations of a c5 t = 8 block spend their time."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P  # noqa: E402

m, w, r, N, sigma = 40000, 5000, 20, 10_000_000, 0.1
_, blk = P.gen_mc_instance(m, w, r, N, sigma, 5)
rho = N / (m * w)
floor = sigma * math.sqrt(rho) * (math.sqrt(m) + math.sqrt(w))
sv = P.McSolver(blk, P.ApgConfig(max_iters=1))
_, tr = sv.step(1, trace=True)
sv.close()
mu_init = tr[0]["mu"] * 0.90 / 0.99
sv = P.McSolver(blk, P.ApgConfig(mu_floor=floor, mu_init=mu_init))
t0 = time.time()
done, tr = sv.step(500, trace=True)
wall = time.time() - t0
print(f"{done} iterations in {wall:.2f} s (lone block)")
tot = sum(t["ms"] for t in tr)
acc = 0.0
for t in tr:
    acc += t["ms"]
    if t["it"] <= 40 or t["it"] % 20 == 0 or t["ms"] > 50:
        print(f"it {t['it']:4d} rank {t['rank']:5d} k {t['k_final']:5d} calls {t['svd_calls']} mu {t['mu']:.3f} rel {t['rel']:.2e} "
              f"ms {t['ms']:8.1f} cum {100 * acc / tot:5.1f}%")
sv.close()
