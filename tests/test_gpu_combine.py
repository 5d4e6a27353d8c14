"""GPU parity of the C-step combiners (P/include/dfc/sketch.hpp) and the D-F-C pipeline
(P/include/dfc/dfc.hpp) against the CPU oracle, plus the reference's exact cases."""
import numpy as np
import pytest

import oracle as O
import paper_1107_0789_b200 as P
from _parity import REL_TOL, cfg_pair, relF, to_oracle_obs

pytestmark = pytest.mark.gpu


def rand_est(rng, m, n, k):
    return P.Estimate(rng.standard_normal((m, k)), rng.standard_normal((n, k)))


def oe(e):
    return O.Estimate(e.left, e.right)


def test_svd_of_product_matches_dense():  # P/tests/test_sketch.cpp:108-118
    rng = np.random.default_rng(0)
    for m, n, k in [(9, 7, 3), (200, 150, 40), (1000, 300, 120), (50, 60, 80), (2000, 900, 300)]:
        l, r = rng.standard_normal((m, k)), rng.standard_normal((n, k))
        est, s = P.svd_of_product(l, r)
        ref = np.linalg.svd(l @ r.T, compute_uv=False)
        assert len(s) == np.sum(ref > 1e-12 * max(m, n) * ref[0])
        assert np.max(np.abs(s - ref[: len(s)])) < 1e-12 * ref[0]
        assert np.linalg.norm(est.dense() - l @ r.T) < 1e-12 * np.linalg.norm(l @ r.T)
    est, s = P.svd_of_product(np.zeros((4, 0)), np.zeros((5, 0)))
    assert est.rank == 0
    with pytest.raises(ValueError):
        P.svd_of_product(np.ones((4, 2)), np.ones((5, 1)))


def test_svd_of_product_rank_deficient():  # numerical-rank truncation (sketch.hpp:82)
    rng = np.random.default_rng(1)
    A = rng.standard_normal((300, 3)) @ rng.standard_normal((3, 40))
    B = rng.standard_normal((200, 40))
    est, s = P.svd_of_product(A, B)
    assert len(s) == 3


def test_column_project_exact_cases():  # P/tests/test_sketch.cpp:184-214
    b0 = P.Estimate(np.array([[1.0], [2.0]]) / np.sqrt(5), np.array([[np.sqrt(5)]]))
    b1 = P.Estimate(np.array([[2.0], [4.0]]) / np.sqrt(20), np.array([[np.sqrt(20)]]))
    proj = P.column_project(b0, [b0, b1], [[0], [1]])
    assert np.linalg.norm(proj.dense() - np.array([[1, 2], [2, 4.0]])) < 1e-12 * 5
    zero = P.Estimate(np.zeros((3, 0)), np.zeros((1, 0)))
    col = P.Estimate(np.ones((3, 1)), np.ones((1, 1)))
    assert P.column_project(zero, [zero, col], [[0], [1]]).rank == 0
    with pytest.raises(ValueError):
        P.column_project(col, [], [])


@pytest.mark.parametrize("t,k", [(3, 5), (8, 12), (4, 40)])
def test_column_project_parity(t, k):
    rng = np.random.default_rng(t * 100 + k)
    m, n = 400, 240
    groups = O.partition_columns(5, 0, n, t)
    blocks = [rand_est(rng, m, len(g), k) for g in groups]
    blocks[1] = P.Estimate(np.zeros((m, 0)), np.zeros((len(groups[1]), 0)))  # a zero-rank block
    for basis in (blocks[0], blocks[2]):
        gp = P.column_project(basis, blocks, groups)
        go = O.column_project(oe(basis), [oe(b) for b in blocks], groups)
        assert relF(gp, go) <= REL_TOL


def test_gen_nystrom_exact_and_parity():  # P/tests/test_sketch.cpp:304-349
    C = P.Estimate(np.array([[1.0], [2.0]]), np.array([[1.0]]))
    R = P.Estimate(np.array([[1.0]]), np.array([[1.0], [2.0]]))
    assert np.linalg.norm(P.gen_nystrom(C, R, [0], [0]).dense() - np.array([[1, 2], [2, 4.0]])) < 1e-12 * 5
    C0 = P.Estimate(np.array([[0.0], [1.0]]), np.array([[1.0]]))
    R0 = P.Estimate(np.array([[1.0]]), np.array([[1.0], [1.0]]))
    assert P.gen_nystrom(C0, R0, [0], [0]).rank == 0
    L = O.gen_low_rank(50, 40, 3, 114, 0)
    rows = np.sort(O.sample_without_replacement(115, 0, 50, 8))
    cols = np.sort(O.sample_without_replacement(116, 0, 40, 8))
    Ch = P.Estimate(L.left, L.right[cols])
    Rh = P.Estimate(L.left[rows], L.right)
    out = P.gen_nystrom(Ch, Rh, rows, cols)
    M = L.dense()
    assert np.linalg.norm(out.dense() - M) < 1e-9 * np.linalg.norm(M)
    rng = np.random.default_rng(3)
    m, n, d, l = 500, 400, 60, 50
    rows = np.sort(rng.choice(m, d, replace=False))
    cols = np.sort(rng.choice(n, l, replace=False))
    Ch, Rh = rand_est(rng, m, l, 12), rand_est(rng, d, n, 9)
    assert relF(P.gen_nystrom(Ch, Rh, rows, cols), O.gen_nystrom(oe(Ch), oe(Rh), rows, cols)) <= REL_TOL
    with pytest.raises(IndexError):
        P.gen_nystrom(P.Estimate(np.ones((3, 1)), np.ones((2, 1))), P.Estimate(np.ones((1, 1)), np.ones((4, 1))),
                      [5], [0, 1])


def test_average_estimates_cases_and_parity():  # P/tests/test_sketch.cpp:360-397
    L = O.gen_low_rank(6, 5, 2, 116, 0)
    Lp = P.Estimate(L.left, L.right)
    assert np.linalg.norm(P.average_estimates([Lp, Lp, Lp]).dense() - L.dense()) < 1e-12 * np.linalg.norm(L.dense())
    assert np.linalg.norm(P.average_estimates([Lp, P.Estimate(L.left, -L.right)]).dense()) < 1e-12
    with pytest.raises(ValueError):
        P.average_estimates([])
    rng = np.random.default_rng(4)
    ests = [rand_est(rng, 300, 200, k) for k in (20, 30, 25, 40)]
    for rc in (None, 10, 50):
        assert relF(P.average_estimates(ests, rc), O.average_estimates([oe(e) for e in ests], rc)) <= REL_TOL
    big = [rand_est(rng, 80, 60, 30) for _ in range(3)]  # total k 90 > min(m, n): compaction path
    assert relF(P.average_estimates(big), O.average_estimates([oe(e) for e in big])) <= REL_TOL


def test_random_project_exact_and_parity():  # P/tests/test_sketch.cpp:246-292
    L = O.gen_low_rank(12, 9, 2, 110, 0)
    M = L.dense()
    groups = [np.arange(0, 3), np.arange(3, 6), np.arange(6, 9)]
    blocks = [O.compact_svd_estimate(M[:, g]) for g in groups]
    pb = [P.Estimate(b.left, b.right) for b in blocks]
    Y = P.random_project(pb, groups, 2, 5, 2, 111, 0)
    assert np.linalg.norm(Y.dense() - M) < 1e-8 * np.linalg.norm(M)
    rng = np.random.default_rng(5)
    groups = O.partition_columns(9, 0, 300, 4)
    blocks = [rand_est(rng, 350, len(g), 15) for g in groups]
    gp = P.random_project(blocks, groups, 20, 5, 2, 77, 3)
    go = O.random_project([oe(b) for b in blocks], groups, 20, 5, 2, 77, 3)
    assert relF(gp, go) <= REL_TOL
    with pytest.raises(ValueError):
        P.random_project([P.Estimate(np.ones((4, 1)), np.ones((4, 1)))], [np.arange(4)], 2, 5, 2, 1, 0)


@pytest.mark.parametrize("variant,ens,kw", [
    ("proj", False, dict(t=3)),
    ("proj", True, dict(t=3)),
    ("rp", False, dict(t=3)),
    ("rp", True, dict(t=2)),
    ("nys", False, dict(l=60, d=60)),
    ("nys", True, dict(l=70, d=50)),
])
def test_dfc_run_parity(variant, ens, kw):
    L0, obs = P.gen_mc_instance(200, 200, 3, 16000, 0.1, 1)
    pc, oc = cfg_pair()
    eo, io = O.dfc_run(to_oracle_obs(obs), variant, ensemble=ens, solver_cfg=oc, seed=1, **kw)
    ep, ip = P.dfc_run(obs, variant, ensemble=ens, solver_cfg=pc, seed=1, workers=2, **kw)
    assert [s.iterations for s in ip["subproblems"]] == [s.iterations for s in io["subproblems"]]
    assert [s.rank for s in ip["subproblems"]] == [s.rank for s in io["subproblems"]]
    assert ep.rank == eo.rank
    assert relF(ep, eo) <= REL_TOL
    assert ip["chosen_k"] == io["chosen_k"] and ip["rank_deficient"] == io["rank_deficient"]


@pytest.mark.parametrize("anchors", [1, 4])
def test_dfc_proj_ens_anchor_parity(anchors):
    """BASELINE c5's "ensemble of 4" (an extension of dfc.hpp:189-195): Proj-Ens anchored on the
    first A plan groups, GPU against the oracle extension."""
    L0, obs = P.gen_mc_instance(200, 200, 3, 16000, 0.1, 1)
    pc, oc = cfg_pair()
    eo, io = O.dfc_run(to_oracle_obs(obs), "proj", ensemble=True, t=6, solver_cfg=oc, seed=1,
                       ensemble_anchors=anchors)
    ep, ip = P.dfc_run(obs, "proj", ensemble=True, t=6, solver_cfg=pc, seed=1, workers=3,
                       ensemble_anchors=anchors)
    assert [s.iterations for s in ip["subproblems"]] == [s.iterations for s in io["subproblems"]]
    assert ep.rank == eo.rank
    assert relF(ep, eo) <= REL_TOL
    with pytest.raises(ValueError):
        P.dfc_run(obs, "rp", ensemble=True, t=3, ensemble_anchors=2)


def test_dfc_rmf_parity():  # DfcTask RMF path (P/tests/test_dfc.cpp:304-320 shape)
    L0, S0, M = P.gen_rmf_instance(60, 72, 2, 200, 0.01, 3)
    r, c = np.meshgrid(np.arange(60), np.arange(72), indexing="ij")
    obs = P.Observed(60, 72, r.T.ravel().astype(np.int64), c.T.ravel().astype(np.int64), M.T.ravel().copy())
    pc, oc = cfg_pair(rel_tol=1e-6, max_iters=2000)
    eo, io = O.dfc_run(to_oracle_obs(obs), "proj", ensemble=True, t=2, seed=5, solver_cfg=oc, task="rmf")
    ep, ip = P.dfc_run(obs, "proj", ensemble=True, t=2, seed=5, solver_cfg=pc, task="rmf")
    assert [s.iterations for s in ip["subproblems"]] == [s.iterations for s in io["subproblems"]]
    assert relF(ep, eo) <= REL_TOL


def test_dfc_empty_blocks_and_errors():  # P/tests/test_dfc.cpp:81-97, 146-161
    obs = P.Observed(3, 4, np.array([0]), np.array([0]), np.array([5.0]))
    est, info = P.dfc_run(obs, "proj", ensemble=True, t=4, seed=2)
    assert est.left.shape[0] == 3 and est.right.shape[0] == 4
    assert np.all(np.isfinite(est.dense()))
    assert sum(s.iterations == 0 for s in info["subproblems"]) == 3
    r, c = np.meshgrid(np.arange(4), np.arange(4), indexing="ij")
    ones = P.Observed(4, 4, r.T.ravel().astype(np.int64), c.T.ravel().astype(np.int64), np.ones(16))
    for bad in (dict(t=0), dict(t=5), dict(t=2, workers=0)):
        with pytest.raises(ValueError):
            P.dfc_run(ones, "proj", **bad)
    for l, d in ((0, 2), (6, 2), (2, 0), (2, 5)):
        with pytest.raises(ValueError):
            P.dfc_run(ones, "nys", l=l, d=d)


def test_dfc_block_failure_carries_index():  # P/tests/test_dfc.cpp:118-144: a failing block -> BlockError
    r, c = np.meshgrid(np.arange(6), np.arange(5), indexing="ij")
    obs = P.Observed(6, 5, r.T.ravel().astype(np.int64), c.T.ravel().astype(np.int64), np.ones(30))
    # an invalid solver config makes every block fail; the lowest index must be reported
    with pytest.raises(P.BlockError) as ei:
        P.dfc_run(obs, "proj", t=2, seed=9, workers=2, solver_cfg=P.ApgConfig(rel_tol=2.0))
    assert ei.value.block == 0 and "block 0" in str(ei.value)


def test_dfc_worker_invariance_bitwise():  # P/tests/test_dfc.cpp:322-342
    L0, obs = P.gen_mc_instance(40, 40, 2, 1600, 0.0, 4)
    for variant, kw in (("proj", dict(t=4)), ("rp", dict(t=4)), ("nys", dict(l=10, d=10))):
        a, _ = P.dfc_run(obs, variant, ensemble=True, seed=11, workers=1, **kw)
        b, _ = P.dfc_run(obs, variant, ensemble=True, seed=11, workers=4, **kw)
        assert np.array_equal(a.left, b.left) and np.array_equal(a.right, b.right)


def test_experiment_harness_matches_oracle():
    """run_experiment on the GPU path (bench.hpp:158-336): per-seed RMSE of every method equal to
    the oracle's dfc_run / apg_mc / F-step-only estimate on the same seeds, summary rows appended."""
    import io

    from paper_1107_0789_b200.experiment import ExperimentSpec, run_experiment, write_csv

    spec = ExperimentSpec(m=100, n=90, r=3, s=4000, sigma=0.1, methods=["base", "part", "proj", "nys", "rp"],
                          seeds=[1, 2], t=3, l_frac=0.3, d_frac=0.3)
    rows = run_experiment(spec)
    assert [r.method for r in rows[-10:]] == sorted(m + s for m in spec.methods for s in ("_mean", "_std"))
    for r in rows[:-10]:
        L0, obs = O.gen_mc_instance(100, 90, 3, 4000, 0.1, r.seed, 0)
        if r.method == "base":
            est, _ = O.apg_mc(obs)
        elif r.method == "part":
            groups = O.partition_columns(r.seed, 0xDFC0000000000001, 90, 3)
            ests = [O.apg_mc(O.extract_columns(obs, g))[0] for g in groups]
            left = np.hstack([e.left for e in ests])
            right = np.zeros((90, left.shape[1]))
            at = 0
            for e, g in zip(ests, groups):
                right[np.asarray(g), at:at + e.rank] = e.right
                at += e.rank
            est = O.Estimate(left, right)
        else:
            est, _ = O.dfc_run(obs, r.method, t=3, l=27, d=30, rp_p=5, rp_q=2, seed=r.seed)
        ref = O.rmse(L0, est)
        assert abs(r.rmse - ref) <= 1e-6 * ref, (r.method, r.seed, r.rmse, ref)
    buf = io.StringIO()
    write_csv(buf, rows)
    assert len(buf.getvalue().splitlines()) == len(rows) + 1
