"""Quick GPU-vs-oracle diagnostics (development aid; the real gates are tests/ -m gpu)."""
import sys, time, traceback
import numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1107_0789_b200 as P
import oracle as O

def rel(a, b):
    A, B = a.dense(), b.dense()
    return np.linalg.norm(A - B) / max(np.linalg.norm(B), 1e-300)

def to_o(obs):
    return O.Observed(obs.m, obs.n, obs.rows, obs.cols, obs.vals)

def cfgs(**kw):
    return P.ApgConfig(**kw), O.apg_cfg(**kw)

def run(name, f):
    t0 = time.time()
    try:
        f()
        print(f"[ok] {name} {time.time()-t0:.2f}s", flush=True)
    except Exception:
        print(f"[FAIL] {name}", flush=True)
        traceback.print_exc()

def t_svdprod():
    rng = np.random.default_rng(0)
    for (m, n, k) in [(9, 7, 3), (200, 150, 40), (1000, 300, 120), (50, 60, 80), (2000, 900, 300)]:
        l = rng.standard_normal((m, k)); r = rng.standard_normal((n, k))
        est, s = P.svd_of_product(l, r)
        ref = np.linalg.svd(l @ r.T, compute_uv=False)
        print(f"   svd_of_product {m}x{n}x{k}: rank {len(s)} vs {np.sum(ref > 1e-12*max(m,n)*ref[0])}, "
              f"s err {np.max(np.abs(s - ref[:len(s)]))/ref[0]:.2e}, recon {np.linalg.norm(est.dense() - l@r.T)/np.linalg.norm(l@r.T):.2e}")

def t_mc(m, n, r, s, sigma, seed, **kw):
    L0, obs = P.gen_mc_instance(m, n, r, s, sigma, seed)
    pc, oc = cfgs(**kw)
    t0 = time.time(); eo, ro = O.apg_mc(to_o(obs), oc); to = time.time() - t0
    t0 = time.time(); ep, rp = P.apg_mc(obs, pc); tp = time.time() - t0
    mism = [ (a['it'], a['rank'], b['rank'], a['k_final'], b['k_final'], a['svd_calls'], b['svd_calls'])
             for a, b in zip(rp.trace, ro.trace) if (a['rank'], a['k_final'], a['svd_calls']) != (b['rank'], b['k_final'], b['svd_calls'])]
    rels = [abs(a['rel'] - b['rel']) / max(abs(b['rel']), 1e-300) for a, b in zip(rp.trace, ro.trace)]
    print(f"   mc {m}x{n} r{r} s{s}: iters gpu {rp.iterations} cpu {ro.iterations}, rank {rp.rank}/{ro.rank}, "
          f"relF {rel(ep, eo):.2e}, obj {rp.objective:.6g}/{ro.objective:.6g}, max rel-trace diff {max(rels) if rels else 0:.1e}, "
          f"trace mismatches {mism[:5]}, t gpu {tp:.2f}s cpu {to:.2f}s")

def t_rmf(m, n, r, s, sigma, seed, **kw):
    L0, S0, M = P.gen_rmf_instance(m, n, r, s, sigma, seed)
    pc, oc = cfgs(**kw)
    lam = O.default_rmf_lambda(m, n)
    eo, so, ro = O.apg_rmf(M, lam, oc)
    ep, sp, rp = P.apg_rmf(M, lam, pc)
    So = np.zeros((m, n)); So[so[0], so[1]] = so[2]
    Sp = np.zeros((m, n)); Sp[sp[0], sp[1]] = sp[2]
    print(f"   rmf {m}x{n}: iters {rp.iterations}/{ro.iterations}, rank {rp.rank}/{ro.rank}, relF L {rel(ep, eo):.2e}, "
          f"relF S {np.linalg.norm(Sp-So)/max(np.linalg.norm(So),1e-300):.2e}, nnzS {len(sp[2])}/{len(so[2])}")

def t_dfc(variant, ens, m, n, r, s, sigma, seed, **kw):
    L0, obs = P.gen_mc_instance(m, n, r, s, sigma, seed)
    pc, oc = cfgs(**kw.pop('cfg', {}))
    eo, io = O.dfc_run(to_o(obs), variant, ensemble=ens, solver_cfg=oc, seed=seed, **kw)
    ep, ip = P.dfc_run(obs, variant, ensemble=ens, solver_cfg=pc, seed=seed, **kw)
    print(f"   dfc {variant} ens={ens} {m}x{n}: relF {rel(ep, eo):.2e}, ranks {ep.rank}/{eo.rank}, "
          f"iters {[x.iterations for x in ip['subproblems']]} vs {[x.iterations for x in io['subproblems']]}, "
          f"factor_ms {ip['factor_ms']:.0f}/{io['factor_ms']:.0f}")

run("svd_of_product", t_svdprod)
run("mc dense path 20x20", lambda: t_mc(20, 20, 2, 400, 0.0, 1))
run("mc 30x30 noisy", lambda: t_mc(30, 30, 3, 450, 0.1, 6))
run("mc 100x100 partial", lambda: t_mc(100, 100, 3, 5000, 0.1, 2))
run("mc 500x500 crit3", lambda: t_mc(500, 500, 5, 62500, 0.1, 1, mu_floor=0.1*0.5*(2*np.sqrt(500))))
run("mc 1000x250 c1 block first 40 its", lambda: t_mc(1000, 250, 10, 50000, 0.1, 1, max_iters=40))
run("rmf 40x40", lambda: t_rmf(40, 40, 3, 160, 0.0, 11))
run("rmf 300x300 crit4", lambda: t_rmf(300, 300, 5, 9000, 0.1, 1, mu_floor=0.1*(2*np.sqrt(300))))
run("dfc proj", lambda: t_dfc("proj", False, 200, 200, 3, 16000, 0.1, 1, t=3))
run("dfc proj ens", lambda: t_dfc("proj", True, 200, 200, 3, 16000, 0.1, 1, t=3))
run("dfc nys", lambda: t_dfc("nys", False, 200, 200, 3, 16000, 0.1, 1, l=60, d=60))
run("dfc rp", lambda: t_dfc("rp", False, 200, 200, 3, 16000, 0.1, 1, t=3))
