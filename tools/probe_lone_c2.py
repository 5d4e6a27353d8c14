"""Lone c2 block latency (what one GPU sees at N = 8 with one block each, and the DFC-Nys
subproblems): block 0 (10000 x 1250) run alone for iterations 1..30 untimed, then iterations
31..40 timed per iteration (host wall per iteration, each ends in a device sync) and one profiled
iteration with the per-op-class CUDA-event accounting and launch count."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P  # noqa: E402

L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
groups = P.partition_columns(1, 0xDFC0000000000001, 10000, 8)
blk = P.extract_columns(obs, groups[0])
del obs
sv = P.McSolver(blk)
sv.step(30)
t0 = time.time()
done, tr = sv.step(10, trace=True)
wall = time.time() - t0
print(f"lone c2 block: iterations 31..40 {1e3 * wall / done:.2f} ms/iteration, per-iteration "
      f"{[round(t['ms'], 1) for t in tr]}, ranks {[t['rank'] for t in tr]}", flush=True)
l0 = P.launch_count()
P.prof_enable(True)
sv.step(1)
prof = P.prof_collect()
P.prof_enable(False)
print(f"launches in one iteration: {P.launch_count() - l0}")
tot = 0.0
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    if v["launches"]:
        tot += v["ms"]
        print(f"  {k:12s} ms {v['ms']:7.2f} launches {v['launches']:5d} TF/s {v['flops'] / max(v['ms'], 1e-9) / 1e9:6.2f}")
print(f"  sum of op time {tot:.2f} ms")
sv.close()
