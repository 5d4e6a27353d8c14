"""BASELINE c5 (scaling config) on one GPU: the full 40000 x 40000 instance from the reference
generator (r = 20, 5% observed = 8e7 cells, sigma 0.1; the sparse partial Fisher-Yates keeps the
host memory at O(s)), DFC-Proj partition into t blocks, all blocks solved concurrently for
`its` APG iterations from the start of the solve (default ApgConfig): block-iterations/s and the
rank trajectories."""
import sys, time, os
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1107_0789_b200 as P
t = int(sys.argv[1]) if len(sys.argv) > 1 else 8
its = int(sys.argv[2]) if len(sys.argv) > 2 else 10
m = n = 40000
t0 = time.time()
L0, obs = P.gen_mc_instance(m, n, 20, 80_000_000, 0.1, 1)
print(f"gen {time.time() - t0:.1f}s nnz {obs.count}", flush=True)
t0 = time.time()
groups = P.partition_columns(1, 0xDFC0000000000001, n, t)
blocks = [P.extract_columns(obs, g) for g in groups]
del obs
print(f"divide {time.time() - t0:.1f}s blocks {[b.n for b in blocks[:4]]} nnz {[b.count for b in blocks[:4]]}", flush=True)
solvers = [P.McSolver(b, P.ApgConfig()) for b in blocks]
pool = ThreadPoolExecutor(len(solvers))
t0 = time.time()
outs = list(pool.map(lambda s: s.step(its, trace=True), solvers))
wall = time.time() - t0
tot = sum(d for d, _ in outs)
print(f"{t} blocks x {its} its: {wall:.2f}s -> {tot / wall:.2f} block-it/s", flush=True)
for g, (d, tr) in enumerate(outs[:4]):
    print(f"  block {g}: ranks {[x['rank'] for x in tr]} ms {[round(x['ms']) for x in tr]}", flush=True)
