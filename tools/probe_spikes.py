"""Find host-side stalls: per-iteration host wall vs summed device time of the library's ops."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 60
L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
groups = P.partition_columns(1, 0xDFC0000000000001, 10000, 8)
for g in (1, 2):
    blk = P.extract_columns(obs, groups[g])
    sv = P.McSolver(blk, P.ApgConfig())
    for it in range(1, iters + 1):
        P.prof_enable(True)
        t0 = time.perf_counter()
        sv.step(1)
        wall = 1e3 * (time.perf_counter() - t0)
        pr = P.prof_collect()
        P.prof_enable(False)
        dev = sum(v['ms'] for v in pr.values())
        if wall > 1.8 * dev + 15:
            top = sorted(pr.items(), key=lambda kv: -kv[1]['ms'])[:3]
            print(f"block {g} it {it}: host {wall:.0f} ms, device ops {dev:.0f} ms, top "
                  + ", ".join(f"{k} {v['ms']:.0f}" for k, v in top), flush=True)
    sv.close()
print("done")
