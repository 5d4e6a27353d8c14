"""GPU parity of the F-step base solvers (apg_mc / apg_rmf) against the CPU oracle.

Cases follow the reference's solver tests (P/tests/test_solvers.cpp) and the BASELINE
config shapes at sizes the oracle finishes in seconds; full-size BASELINE blocks are
checked through windows of iterations and size-independent properties.
"""
import numpy as np
import pytest

import oracle as O
import paper_1107_0789_b200 as P
from _parity import assert_mc_parity, assert_rmf_parity, cfg_pair, relF, to_oracle_obs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,r,s,sigma,seed", [
    (20, 20, 2, 400, 0.0, 1),      # fully observed noiseless (test_solvers.cpp:120-129), dense SVT path
    (25, 18, 3, 220, 0.2, 11),     # objective bound cases (:149-157)
    (30, 30, 3, 450, 0.1, 6),      # determinism case (:159-169)
    (15, 15, 2, 150, 0.05, 7),     # report accounting (:186-199)
    (100, 100, 3, 5000, 0.1, 2),   # randomized partial-SVD path (min(m,n) > 64)
    (80, 300, 4, 9000, 0.1, 3),    # wide block (m < n)
    (300, 70, 4, 8000, 0.1, 4),    # tall block, min(m,n) = 70
    (120, 100, 2, 12000, 0.0, 5),  # fully observed exact rank 2 < b: rank-deficient sketches ->
                                   # CholQR breakdown -> Householder fallback in the range finder
    (130, 75, 3, 3000, 0.1, 9),    # ragged 64x64 SDDMM tiles in both directions
])
@pytest.mark.parametrize("op_mode", ["0", "1", "2"], ids=["factored_op", "dense_op", "dense_qr_op"])
def test_apg_mc_parity(m, n, r, s, sigma, seed, op_mode, monkeypatch):
    # every SVT operator form: factored (SDDMM + SpMM + low-rank GEMMs), materialised, and
    # materialised + CholeskyQR2-compressed (m >= n)
    monkeypatch.setenv("DFCG_DENSE_OP", op_mode)
    L0, obs = P.gen_mc_instance(m, n, r, s, sigma, seed)
    assert_mc_parity(obs)


def test_apg_mc_high_accuracy_noiseless():
    """ApgConfig::high_accuracy (rel_tol 1e-9, floor 0) on a noiseless instance; exercises the
    Householder fallback (rank-deficient sketches). Below rel ~ sqrt(2 eps) ~ 2e-8 the stop
    test's cancellation formula (solvers.hpp:190-193) is decided by rounding, so the two
    implementations may stop a few iterations apart; both must reach the same matrix."""
    L0, obs = P.gen_mc_instance(100, 100, 5, 10000, 0.0, 3)
    pc, oc = cfg_pair(max_iters=400, rel_tol=1e-9, mu_decay=0.5, mu_floor=0.0)
    eo, ro = O.apg_mc(to_oracle_obs(obs), oc)
    ep, rp = P.apg_mc(obs, pc)
    # the same rel trajectory while rel is above the formula's noise floor: rel^2 ||L||^2 is a
    # difference of O(||L||^2) terms, so rel carries an absolute rounding error ~ c eps / rel ...
    floor = 1e-7
    for tg, to in zip(rp.trace, ro.trace):
        if to["rel"] < 1e-6:
            break
        assert abs(tg["rel"] - to["rel"]) <= 1e-4 * to["rel"] + 1e-13 / to["rel"], (tg["it"], tg["rel"], to["rel"])
    # ... then both stop on a rounding event inside the noise-floor regime (rel ~ 3e-8)
    first_floor = next(t["it"] for t in ro.trace if t["rel"] < floor)
    assert first_floor <= rp.iterations <= ro.iterations + 10, (rp.iterations, ro.iterations, first_floor)
    assert rp.rank == ro.rank == 5
    assert relF(ep, eo) <= 1e-6
    assert np.linalg.norm(ep.dense() - L0.dense()) / 100.0 < 1e-6


def test_apg_mc_line_search():
    L0, obs = P.gen_mc_instance(120, 90, 3, 4000, 0.1, 5)
    assert_mc_parity(obs, line_search=True)


def test_apg_mc_acceptance_floor_500():  # acceptance criterion 3 setup (P/tests/acceptance.cpp:121-161)
    m = n = 500
    L0, obs = P.gen_mc_instance(m, n, 5, 62500, 0.1, 1)
    ep, rp, eo, ro = assert_mc_parity(obs, mu_floor=0.1 * 0.5 * (2 * np.sqrt(500)))
    assert O.rmse(O.Estimate(L0.left, L0.right), O.Estimate(ep.left, ep.right)) < 0.15


@pytest.mark.parametrize("op_mode", ["0", "1", "2", "auto"])
def test_apg_mc_c1_block_window(op_mode, monkeypatch):  # BASELINE c1 block 1000 x 250, default config, 60 its
    if op_mode != "auto":
        monkeypatch.setenv("DFCG_DENSE_OP", op_mode)
    L0, obs = P.gen_mc_instance(1000, 1000, 10, 200000, 0.1, 1)
    groups = P.partition_columns(1, 0xDFC0000000000001, 1000, 4)
    blk = P.extract_columns(obs, groups[0])
    assert_mc_parity(blk, max_iters=60)


@pytest.mark.parametrize("op_mode", ["0", "1", "2", "auto"])
def test_apg_mc_wide_row_block_window(op_mode, monkeypatch):
    """A DFC-Nys row subproblem (R-hat) shape at c1 scale: 250 x 1000 (m < n), default config,
    60 iterations — the wide operator path (CholeskyQR2 of the transposed dense operator)."""
    if op_mode != "auto":
        monkeypatch.setenv("DFCG_DENSE_OP", op_mode)
    L0, obs = P.gen_mc_instance(1000, 1000, 10, 200000, 0.1, 1)
    rows = np.sort(P.sample_without_replacement(1, 0xDFC0000000000003, 1000, 250))
    assert_mc_parity(P.extract_rows(obs, rows), max_iters=60)


def test_apg_mc_c4_standin_block():
    """A block of the recommender-shaped c4 stand-in (Zipf popularity, integer ratings with a
    3.6 offset: a large rank-one mean component), default config, 60 iterations."""
    m, n = 400, 3000
    groups = P.partition_columns(3, 0xDFC0000000000001, n, 8)
    blk = P.gen_recsys_instance(m, n, 5, 0.05, 3, cols=groups[0])
    assert_mc_parity(blk, max_iters=60)


def test_apg_mc_operator_switching():
    """A sparse block whose rank rises past and falls back below the dense-operator threshold
    (acceptance-style floor, P/tests/acceptance.cpp:127-130): iterations switch between the
    factored and the (compressed) dense operator and back, including the deferred left factors
    of compressed iterations."""
    m, n = 2000, 400
    L0, obs = P.gen_mc_instance(m, n, 10, m * n // 20, 0.1, 13)
    floor = 0.1 * np.sqrt(0.05) * (np.sqrt(m) + np.sqrt(n))
    assert_mc_parity(obs, mu_floor=floor, max_iters=150)


def test_apg_mc_all_zero_observations():  # P/tests/test_solvers.cpp:131-139
    r, c = np.meshgrid(np.arange(4), np.arange(4), indexing="ij")
    obs = P.Observed(4, 4, r.T.ravel().astype(np.int64), c.T.ravel().astype(np.int64), np.zeros(16))
    est, rep = P.apg_mc(obs)
    assert est.rank == 0 and rep.objective == 0.0 and rep.residual == 0.0


def test_apg_mc_validation_errors():  # P/tests/test_solvers.cpp:171-184
    empty = P.Observed(3, 3, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0))
    with pytest.raises(ValueError):
        P.apg_mc(empty)
    one = P.Observed(2, 2, np.array([0]), np.array([0]), np.array([1.0]))
    with pytest.raises(ValueError):
        P.apg_mc(one, P.ApgConfig(rel_tol=0.0))
    with pytest.raises(ValueError):
        P.apg_mc(one, P.ApgConfig(mu_decay=1.0))
    with pytest.raises(ValueError):
        P.apg_mc(one, P.ApgConfig(mu_init=1.0, mu_floor=2.0))
    dup = P.Observed(2, 2, np.array([0, 0]), np.array([0, 0]), np.array([1.0, 2.0]))
    with pytest.raises(ValueError):
        P.apg_mc(dup)
    bad = P.Observed(2, 2, np.array([5]), np.array([0]), np.array([1.0]))
    with pytest.raises(IndexError):
        P.apg_mc(bad)


def test_apg_mc_deterministic_bitwise():  # P/tests/test_solvers.cpp:159-169
    L0, obs = P.gen_mc_instance(120, 100, 3, 6000, 0.1, 8)
    a, ra = P.apg_mc(obs)
    b, rb = P.apg_mc(obs)
    assert ra.iterations == rb.iterations and ra.objective == rb.objective
    assert np.array_equal(a.left, b.left) and np.array_equal(a.right, b.right)


def test_apg_mc_c2_block_properties():
    """BASELINE c2 block (10000 x 1250, 10% observed): the first 9 iterations against the oracle
    (ranks climb to ~500 with a k doubling: iterations 5-9 run the dense and the
    CholeskyQR2-compressed operators at the real block shape; ~1-2 min of oracle time), then 30
    GPU iterations checked through properties (objective bound, residual consistency,
    orthonormal left factor)."""
    m, n = 10000, 1250
    L0, obs = P.gen_mc_instance(m, n, 10, m * n // 10, 0.1, 1)
    assert_mc_parity(obs, max_iters=9)
    est, rep = P.apg_mc(obs, P.ApgConfig(max_iters=30))
    assert rep.iterations == 30
    # residual reported == residual recomputed from the factors on Omega
    vals = np.einsum("ij,ij->i", est.left[obs.rows], est.right[obs.cols])
    res = np.linalg.norm(vals - obs.vals)
    assert abs(res - rep.residual) <= 1e-9 * max(1.0, res)
    # L = 0 is feasible: objective <= 0.5 ||P_Omega M||^2 (P/tests/test_solvers.cpp:149-157)
    assert rep.objective <= 0.5 * float(obs.vals @ obs.vals)
    # left factor = U of an SVT: orthonormal columns
    G = est.left.T @ est.left
    assert np.abs(G - np.eye(G.shape[0])).max() < 1e-10


@pytest.mark.parametrize("m,n,r,s,sigma,seed", [
    (40, 40, 3, 160, 0.0, 11),     # RecoversSparseOutliers (test_solvers.cpp:222-228) shape
    (20, 25, 2, 50, 0.1, 21),      # feasibility cases (:241-250)
    (30, 30, 2, 90, 0.05, 8),      # determinism case (:253-262)
    (120, 90, 3, 1000, 0.05, 4),   # partial-SVD path (min > 64)
])
@pytest.mark.parametrize("op_mode", ["1", "2"], ids=["dense_op", "dense_qr_op"])
def test_apg_rmf_parity(m, n, r, s, sigma, seed, op_mode, monkeypatch):
    # the dense RMF operator as is, and CholeskyQR2-compressed (m >= n)
    monkeypatch.setenv("DFCG_DENSE_OP", op_mode)
    L0, S0, M = P.gen_rmf_instance(m, n, r, s, sigma, seed)
    assert_rmf_parity(M, O.default_rmf_lambda(m, n))


def test_apg_rmf_acceptance_floor_300():  # acceptance criterion 4 setup (P/tests/acceptance.cpp:164-195)
    m = n = 300
    L0, S0, M = P.gen_rmf_instance(m, n, 5, 9000, 0.1, 1)
    assert_rmf_parity(M, O.default_rmf_lambda(m, n), mu_floor=0.1 * 2 * np.sqrt(300))


@pytest.mark.parametrize("op_mode", ["1", "2", "auto"])
def test_apg_rmf_bounded_outliers_c3_shape(op_mode, monkeypatch):  # BASELINE c3 value model (U[-10,10], sigma 0.01), scaled
    if op_mode != "auto":
        monkeypatch.setenv("DFCG_DENSE_OP", op_mode)
    L0, S0, M = P.gen_rmf_instance(400, 100, 4, 4000, 0.01, 3, lo=-10.0, hi=10.0)
    assert_rmf_parity(M, O.default_rmf_lambda(400, 100), max_iters=120)


def test_apg_rmf_line_search_and_edge_cases():
    L0, S0, M = P.gen_rmf_instance(30, 24, 2, 60, 0.05, 2)
    assert_rmf_parity(M, O.default_rmf_lambda(30, 24), line_search=True, max_iters=200)
    spike = np.zeros((10, 12))
    spike[3, 4] = 50.0
    L, S, rep = P.apg_rmf(spike, 0.01, P.ApgConfig(rel_tol=1e-6, max_iters=2000))
    assert L.rank == 0
    Sd = np.zeros_like(spike)
    Sd[S[0], S[1]] = S[2]
    assert np.linalg.norm(Sd - spike) < 1e-3 * 50.0
    L, S, rep = P.apg_rmf(np.zeros((6, 5)), 0.3)
    assert L.rank == 0 and len(S[2]) == 0 and rep.residual == 0.0 and rep.objective == 0.0
    with pytest.raises(ValueError):
        P.apg_rmf(np.ones((3, 3)), 0.0)
    bad = np.ones((3, 3))
    bad[1, 1] = np.nan
    with pytest.raises(ValueError):
        P.apg_rmf(bad, 0.5)
