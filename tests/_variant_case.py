"""Child process of test_gpu_variants.py: one MC parity case (Jacobi block path: b > 64) under
whatever DFCG_* environment the parent set; prints OK or raises."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1107_0789_b200 as P  # noqa: E402
from _parity import assert_mc_parity  # noqa: E402

L0, obs = P.gen_mc_instance(600, 400, 20, 60000, 0.1, 21)
assert_mc_parity(obs, max_iters=12)
print("OK")
