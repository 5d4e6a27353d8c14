import numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_1107_0789_b200 as P
rng = np.random.default_rng(0)
for (m, n, k, scale) in [(200, 150, 20, False), (200, 150, 20, True), (2000, 900, 80, True)]:
    L = rng.standard_normal((m, k)); R = rng.standard_normal((n, k))
    if scale:
        R = R * np.logspace(0, -6, k)
    est = P.svd_of_product(L, R)[0] if isinstance(P.svd_of_product(L, R), tuple) else P.svd_of_product(L, R)
    A = L @ R.T
    B = est.left @ est.right.T
    print(m, n, k, scale, np.linalg.norm(A - B) / np.linalg.norm(A), np.abs(est.left.T @ est.left - np.eye(est.left.shape[1])).max())
