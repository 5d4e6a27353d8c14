"""BASELINE c4 stand-in (recommender-shaped, 17770 x 480189, ~1% observed, Zipf popularity, r = 30,
ratings clip(round(3.6 + A B^T + N(0, 0.8^2)), 1, 5); DFC-Proj t = 64): the first `nb` of the 64
column blocks generated directly (gen_recsys_instance restricted to the block's columns) and solved
concurrently on one GPU for `its` iterations; then one profiled iteration of block 0."""
import sys, time, os, json
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 8
its = int(sys.argv[2]) if len(sys.argv) > 2 else 30
m, n, r, dens = 17770, 480189, 30, 0.0117
t0 = time.time()
groups = P.partition_columns(1, 0xDFC0000000000001, n, 64)
blocks = [P.gen_recsys_instance(m, n, r, dens, 1, cols=groups[g]) for g in range(nb)]
print(f"gen {time.time() - t0:.1f}s  nnz per block {[b.count for b in blocks]}", flush=True)
solvers = [P.McSolver(b, P.ApgConfig()) for b in blocks]
pool = ThreadPoolExecutor(nb)
t0 = time.time()
outs = list(pool.map(lambda s: s.step(its, trace=True), solvers))
wall = time.time() - t0
tot = sum(d for d, _ in outs)
print(f"{nb} blocks x {its} its: {wall:.2f}s -> {tot / wall:.1f} block-it/s", flush=True)
for g, (d, tr) in enumerate(outs):
    print(f"  block {g}: ranks {[t['rank'] for t in tr[::5]]} last ms {[round(t['ms'], 1) for t in tr[-3:]]}", flush=True)
P.prof_enable(True)
solvers[0].step(1)
prof = P.prof_collect()
P.prof_enable(False)
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    if v["launches"]:
        print(f"  {k:12s} ms {v['ms']:.2f} launches {v['launches']} GB/s {v['bytes'] / max(v['ms'], 1e-9) / 1e6:.0f} "
              f"TF/s {v['flops'] / max(v['ms'], 1e-9) / 1e9:.2f}", flush=True)
