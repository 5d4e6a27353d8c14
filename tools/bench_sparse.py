"""Microbenchmark of the APG-MC iteration's sparse kernels (dfcg_bench_sparse): forward SpMM R X,
transposed SpMM R^T Q and the SDDMM residual; the segmented-gather SpMM / tiled SDDMM ("gather"),
the slab kernels ("slab") and the cache-blocked (chunked) gather SpMM ("chunked"), on the c5 block (40000 x 5000, N = 1e7) and the c2
block (10000 x 1250, N ~ 1.25e6) at their low-rank sketch widths. Rates are algorithmic bytes
(the same accounting as the per-op profile) per CUDA-event time; sums compare the two modes."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1107_0789_b200 as P  # noqa: E402
from paper_1107_0789_b200 import _lib as L  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cases = []
L0, blk = P.gen_mc_instance(40000, 5000, 20, 10_000_000, 0.1, 5)
cases.append(("c5 block 40000x5000", blk, 35, 20))
L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
g = P.partition_columns(1, 0xDFC0000000000001, 10000, 8)
cases.append(("c2 block 10000x1250", P.extract_columns(obs, g[0]), 25, 10))
del obs
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0) \
    if os.path.exists("MEASURED_PEAKS.json") else 6650.0
out = []
for name, o, b, kY in cases:
    keep = L._Keep()
    oc = L._obs_in(o, keep)
    N, m, n = o.count, o.m, o.n
    by = {"spmm": 12.0 * N + 8.0 * b * (n + m), "spmm_t": 12.0 * N + 8.0 * b * (m + n),
          "sddmm": 24.0 * N + 8.0 * (m + n) * kY}
    res = {}
    # (spmm mode, sddmm mode): 0 = gather SpMM / tiled SDDMM, 1 = slab kernels, 2 = chunked SpMM
    for key, (ms_mode, sd_mode) in {"gather": (0, 0), "slab": (1, 1), "chunked": (2, 0), "gather16": (3, 0), "chunked16": (4, 0), "wide": (5, 0)}.items():
        ms = (C.c_double * 3)()
        sm = (C.c_double * 3)()
        L._check(L.lib().dfcg_bench_sparse(L.context(0), C.byref(oc), C.c_int64(b), C.c_int64(kY), C.c_int32(reps),
                                           C.c_int32(ms_mode), C.c_int32(sd_mode), ms, sm))
        res[key] = (list(ms), list(sm))
    row = dict(case=name, N=N, b=b, kY=kY)
    for i, k in enumerate(("spmm", "spmm_t", "sddmm")):
        row[k] = {}
        for key in res:
            t_ms = res[key][0][i]
            row[k][key] = dict(us=round(1e3 * t_ms, 1), gbs=round(by[k] / (t_ms * 1e-3) / 1e9, 1),
                               frac=round(by[k] / (t_ms * 1e-3) / 1e9 / peak, 3),
                               sum_rel_diff=abs(res[key][1][i] - res["gather"][1][i]) / max(abs(res["gather"][1][i]), 1e-300))
    out.append(row)
    print(json.dumps(row), flush=True)
