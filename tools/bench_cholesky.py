"""Microbenchmark of the CholeskyQR Cholesky + inverse (dfcg_bench_cholesky) at the c2 sizes
(n = 720: the range finder's b; n = 1250: the CholeskyQR2 of the dense operator): the fused
cooperative kernel at several CTA counts (DFCG_CHOL_P) against the launch-per-panel path
(DFCG_CHOL_FUSED=0). Each configuration runs in its own process (the switches are read once)."""
import ctypes as C
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    from paper_1107_0789_b200 import _lib as L

    n, inv = int(sys.argv[2]), int(sys.argv[3])
    ms, rr, ir = C.c_double(), C.c_double(), C.c_double()
    L._check(L.lib().dfcg_bench_cholesky(L.context(0), C.c_int64(n), C.c_int32(20), C.c_int32(inv), C.byref(ms),
                                         C.byref(rr), C.byref(ir)))
    print(json.dumps(dict(n=n, inverse=inv, ms=round(ms.value, 4), relres=rr.value, invres=ir.value)))
    sys.exit(0)

sweep = os.environ.get("CHOL_BENCH_P", "8,12,16,32,64,148")
configs = [("per-panel", {"DFCG_CHOL_FUSED": "0"})] + \
          [(f"fused P={p}", {"DFCG_CHOL_FUSED": "1", "DFCG_CHOL_P": p}) for p in sweep.split(",") if p] + \
          [("fused default P", {"DFCG_CHOL_FUSED": "1"})]
for n in [int(x) for x in os.environ.get("CHOL_BENCH_N", "720,1250").split(",")]:
    for inv in (1, 0):
        for name, env in configs:
            try:
                r = subprocess.run([sys.executable, __file__, "--one", str(n), str(inv)], env={**os.environ, **env},
                                   capture_output=True, text=True, timeout=int(os.environ.get("CHOL_BENCH_TIMEOUT", "120")))
                line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else f"failed: {r.stderr[-300:]}"
            except subprocess.TimeoutExpired:
                line = "timed out"
            print(f"{name:18s} {line}", flush=True)
