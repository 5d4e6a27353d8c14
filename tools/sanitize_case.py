"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): every kernel family
of the hot path on small shapes — apg_mc (factored operator: slab SDDMM / SpMM, small Jacobi),
apg_mc on a dense-operator shape (CholeskyQR2, resident Jacobi rounds), apg_rmf, and dfc_run
DFC-Proj / Proj-Ens / Nys / RP (combiners)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1107_0789_b200 as P  # noqa: E402

L0, obs = P.gen_mc_instance(160, 120, 3, 6000, 0.1, 7)
est, rep = P.apg_mc(obs, P.ApgConfig(max_iters=15))
print("apg_mc factored", rep.iterations, rep.rank, flush=True)
L0, obs2 = P.gen_mc_instance(300, 140, 4, 30000, 0.1, 3)
est, rep = P.apg_mc(obs2, P.ApgConfig(max_iters=6))
print("apg_mc dense-operator shape", rep.iterations, rep.rank, flush=True)
L0, S0, M = P.gen_rmf_instance(120, 90, 2, 500, 0.01, 3)
est, S, rep = P.apg_rmf(np.asfortranarray(M), 1.0 / np.sqrt(120), P.ApgConfig(max_iters=8))
print("apg_rmf", rep.iterations, rep.rank, flush=True)
cfg = P.ApgConfig(max_iters=8)
for variant, kw in (("proj", dict(t=3)), ("proj", dict(t=3, ensemble=True)), ("nys", dict(l=40, d=50)),
                    ("rp", dict(t=3))):
    e, info = P.dfc_run(obs, variant, seed=2, workers=2, solver_cfg=cfg, **kw)
    print("dfc_run", variant, kw, e.rank, flush=True)
print("SANITIZE CASE DONE")
