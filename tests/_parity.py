"""Shared helpers for GPU-vs-oracle parity tests (tolerances per north_star: FP64, relative
Frobenius error <= 1e-6 on L-hat and S-hat, identical iteration counts)."""
import numpy as np

import oracle as O
import paper_1107_0789_b200 as P

REL_TOL = 1e-6


def relF(a, b):
    A, B = a.dense(), b.dense()
    nb = np.linalg.norm(B)
    if nb == 0.0:
        return float(np.linalg.norm(A))
    return float(np.linalg.norm(A - B) / nb)


def to_oracle_obs(obs):
    return O.Observed(obs.m, obs.n, obs.rows, obs.cols, obs.vals)


def cfg_pair(**kw):
    return P.ApgConfig(**kw), O.apg_cfg(**kw)


def dense_S(trip, m, n):
    S = np.zeros((m, n))
    S[trip[0], trip[1]] = trip[2]
    return S


def assert_mc_parity(obs, **kw):
    pc, oc = cfg_pair(**kw)
    eo, ro = O.apg_mc(to_oracle_obs(obs), oc)
    ep, rp = P.apg_mc(obs, pc)
    assert rp.iterations == ro.iterations, (rp.iterations, ro.iterations)
    assert rp.rank == ro.rank, (rp.rank, ro.rank)
    assert [t["rank"] for t in rp.trace] == [t["rank"] for t in ro.trace]
    assert [t["k_final"] for t in rp.trace] == [t["k_final"] for t in ro.trace]
    assert relF(ep, eo) <= REL_TOL, relF(ep, eo)
    assert abs(rp.objective - ro.objective) <= REL_TOL * max(1.0, abs(ro.objective))
    assert abs(rp.residual - ro.residual) <= REL_TOL * max(1.0, abs(ro.residual))
    return ep, rp, eo, ro


def assert_rmf_parity(M, lam, **kw):
    pc, oc = cfg_pair(**kw)
    eo, so, ro = O.apg_rmf(M, lam, oc)
    ep, sp, rp = P.apg_rmf(M, lam, pc)
    m, n = M.shape
    assert rp.iterations == ro.iterations, (rp.iterations, ro.iterations)
    assert rp.rank == ro.rank
    assert relF(ep, eo) <= REL_TOL, relF(ep, eo)
    So, Sp = dense_S(so, m, n), dense_S(sp, m, n)
    nS = np.linalg.norm(So)
    assert (np.linalg.norm(Sp - So) / nS if nS > 0 else np.linalg.norm(Sp)) <= REL_TOL
    return ep, sp, rp, eo, so, ro
