"""Where the c2 e2e solve time goes: the 8 blocks solved concurrently (one thread + stream each,
as bench.py's e2e does), per-iteration host wall times aggregated over iteration windows."""
import sys, time, os
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1107_0789_b200 as P
L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
groups = P.partition_columns(1, 0xDFC0000000000001, 10000, 8)
blocks = [P.extract_columns(obs, g) for g in groups]
pool = ThreadPoolExecutor(8)
P.apg_mc(blocks[0], P.ApgConfig(max_iters=2))  # context + normal cache warm
for rep_i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    t0 = time.time()
    outs = list(pool.map(lambda b: (time.time(), P.apg_mc(b, P.ApgConfig()), time.time()), blocks))
    wall = time.time() - t0
    print(f"run {rep_i}: wall {wall:.2f}s", flush=True)
edges = [0, 10, 30, 100, 200, 300, 400, 500]
for g, (ts, (est, rep), te) in enumerate(outs):
    ms = np.array([t["ms"] for t in rep.trace])
    win = [ms[a:b].sum() / 1e3 for a, b in zip(edges[:-1], edges[1:])]
    print(f"block {g}: its {rep.iterations} start {ts - t0:.2f} end {te - t0:.2f} setup {(te - ts) - ms.sum() / 1e3:.2f}s "
          f"windows " + " ".join(f"{w:.2f}" for w in win) + f" | retries {sum(t['svd_calls'] > 1 for t in rep.trace)}"
          f" dense {sum(t['k_final'] == 0 for t in rep.trace)}", flush=True)
