"""One launch set of the sparse kernels at the c5 block (40000 x 5000, N = 1e7, b = 35) for ncu:
gather SpMM / tiled SDDMM (mode 0) then the chunked SpMM plan (mode 2)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P  # noqa: E402
from paper_1107_0789_b200 import _lib as L  # noqa: E402

_, blk = P.gen_mc_instance(40000, 5000, 20, 10_000_000, 0.1, 5)
keep = L._Keep()
oc = L._obs_in(blk, keep)
for mode in (0, 2):
    ms = (C.c_double * 3)()
    sm = (C.c_double * 3)()
    L._check(L.lib().dfcg_bench_sparse(L.context(0), C.byref(oc), C.c_int64(35), C.c_int64(20), C.c_int32(1),
                                       C.c_int32(mode), C.c_int32(0), ms, sm))
    print(mode, list(ms))
