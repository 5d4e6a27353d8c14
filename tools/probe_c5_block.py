"""One BASELINE c5-shaped block (40000 x 5000 = a t = 8 column block of the 40k x 40k instance:
r = 20, 5% observed -> N = 1e7, sigma = 0.1; generated directly at block shape with the reference
generator, statistically the same as a column block) in its low-rank regime: acceptance-style
floor, iterations 1..skip unprofiled, then a profiled window with per-op algorithmic rates — the
SDDMM / SpMM at 8x the c2 block's nnz."""
import sys, time, os, json, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P
skip = int(sys.argv[1]) if len(sys.argv) > 1 else 60
win = int(sys.argv[2]) if len(sys.argv) > 2 else 10
m, w, r, s, sigma = 40000, 5000, 20, 10_000_000, 0.1
t0 = time.time()
L0, blk = P.gen_mc_instance(m, w, r, s, sigma, 5)
print(f"gen {time.time() - t0:.1f}s nnz {blk.count}", flush=True)
floor = sigma * math.sqrt(s / (m * w)) * (math.sqrt(m) + math.sqrt(w))
sv = P.McSolver(blk, P.ApgConfig(mu_floor=floor))
t0 = time.time()
done, tr = sv.step(skip, trace=True)
print(f"iterations 1..{done}: {time.time() - t0:.2f}s ranks {[t['rank'] for t in tr[::10]]} last {tr[-1]['rank']}",
      flush=True)
P.prof_enable(True)
t0 = time.time()
done, tr = sv.step(win, trace=True)
wall = time.time() - t0
prof = P.prof_collect()
P.prof_enable(False)
print(f"window {done} its: {1e3 * wall / max(done, 1):.2f} ms/it, rank {tr[-1]['rank'] if tr else None}", flush=True)
out = {}
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    if v["launches"]:
        out[k] = dict(ms_per_it=round(v["ms"] / max(done, 1), 3), launches=v["launches"],
                      us_per_launch=round(1e3 * v["ms"] / v["launches"], 1),
                      gbs=round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1),
                      tflops=round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 2))
        print(f"  {k:12s} {out[k]}", flush=True)
print(json.dumps(dict(floor=floor, window=[skip + 1, skip + done], per_op=out)))
