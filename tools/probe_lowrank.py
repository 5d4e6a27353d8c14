"""c2 block under the acceptance-style floor (P/tests/acceptance.cpp:127-130: mu_floor =
sigma sqrt(rho) (sqrt(m) + sqrt(w))): the late, low-rank regime where SDDMM / SpMM are
HBM-bound. Prints the trajectory and the per-op rates of a late window."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P

skip = int(sys.argv[1]) if len(sys.argv) > 1 else 60
win = int(sys.argv[2]) if len(sys.argv) > 2 else 20
m, n, w = 10000, 10000, 1250
L0, obs = P.gen_mc_instance(m, n, 10, 10_000_000, 0.1, 1)
groups = P.partition_columns(1, 0xDFC0000000000001, n, 8)
blk = P.extract_columns(obs, groups[0])
floor = 0.1 * math.sqrt(0.1) * (math.sqrt(m) + math.sqrt(w))
cfg = P.ApgConfig(mu_floor=floor)
sv = P.McSolver(blk, cfg)
t0 = time.perf_counter()
sv.step(skip)
print(f"floor {floor:.3f}: first {skip} iterations {time.perf_counter() - t0:.2f}s", flush=True)
P.prof_enable(True)
t0 = time.perf_counter()
done, tr = sv.step(win, trace=True)
wall = time.perf_counter() - t0
prof = P.prof_collect()
P.prof_enable(False)
est, rep = sv.finish()
print(f"window {done} iterations {wall * 1e3:.1f} ms ({wall * 1e3 / max(done, 1):.2f} ms/it), rank {rep.rank}, "
      f"total iterations {rep.iterations}")
print("ranks", [t['rank'] for t in tr], "k", [t['k_final'] for t in tr])
tot = sum(v['ms'] for v in prof.values())
for op, v in sorted(prof.items(), key=lambda kv: -kv[1]['ms']):
    if v['launches'] == 0:
        continue
    tf = v['flops'] / (v['ms'] * 1e-3) / 1e12 if v['ms'] else 0
    gb = v['bytes'] / (v['ms'] * 1e-3) / 1e9 if v['ms'] else 0
    print(f"{op:12s} launches {v['launches']:6d} ms {v['ms']:8.2f} ({100 * v['ms'] / tot:5.1f}%) {tf:6.2f} TFLOP/s "
          f"{gb:8.1f} GB/s")
sv.close()
