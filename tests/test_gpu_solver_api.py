"""GPU checks of the resumable solver ABI (dfcg_mc_solver_*), the per-block projection used by
the multi-GPU combine, and the multi-rank bench path (ranks sharing one GPU over gloo)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
import paper_1107_0789_b200 as P
from _parity import REL_TOL, relF

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_stepped_solver_equals_one_shot_bitwise():
    L0, obs = P.gen_mc_instance(150, 120, 3, 8000, 0.1, 9)
    ref, rref = P.apg_mc(obs)
    sv = P.McSolver(obs)
    total = 0
    while True:
        k = sv.step(7)
        total += k
        if k < 7:
            break
    est, rep = sv.finish()
    sv.close()
    assert total == rref.iterations == rep.iterations
    assert np.array_equal(est.left, ref.left) and np.array_equal(est.right, ref.right)
    assert rep.objective == rref.objective


def test_stepped_solver_matches_oracle_window():
    L0, obs = P.gen_mc_instance(300, 100, 4, 9000, 0.1, 2)
    sv = P.McSolver(obs, P.ApgConfig())
    done, tr = sv.step(25, trace=True)
    est, rep = sv.finish()
    sv.close()
    eo, ro = O.apg_mc(O.Observed(obs.m, obs.n, obs.rows, obs.cols, obs.vals), O.apg_cfg(max_iters=25))
    assert done == ro.iterations
    assert [t["rank"] for t in tr] == [t["rank"] for t in ro.trace]
    assert relF(est, eo) <= REL_TOL


def test_project_block_matches_formula():
    rng = np.random.default_rng(7)
    Ub, _ = np.linalg.qr(rng.standard_normal((400, 30)))
    blk = P.Estimate(rng.standard_normal((400, 12)), rng.standard_normal((90, 12)))
    got = P.project_block(Ub, blk)
    want = blk.right @ (Ub.T @ blk.left).T
    assert np.abs(got - want).max() < 1e-12 * np.abs(want).max()
    zero = P.Estimate(np.zeros((400, 0)), np.zeros((90, 0)))
    assert np.all(P.project_block(Ub, zero) == 0.0)


def test_bench_multi_rank_path_on_one_gpu():
    """torchrun with 2 ranks sharing the GPU (DFCG_DIST_BACKEND=gloo): sharding, combine
    (basis broadcast + row gather) and the JSON contract on the small c1 workload."""
    env = dict(os.environ, DFCG_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--workload", "c1", "--steps", "2", "--warmup", "1", "--prologue", "2", "--no-cpu"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["gpu_launches"] > 0
    assert sorted(set(line["e2e"]["owner"])) == [0, 1]  # LPT shares: both ranks solve blocks


def test_device_normal_stream_matches_reference_rng():
    """The SVT's Gaussian draws (SeededRng(0x737674, 0|1), P/include/dfc/rng.hpp:62-66): raw
    mt19937_64 words drawn on the host (bit-identical), Box-Muller on the device with CUDA's
    log / cos — within a few ulp of the host libm values the oracle uses, across chunk
    boundaries (4 Mi normals per chunk)."""
    import ctypes as C

    L = P.lib()
    for stream in (0, 1):
        for pos, n in ((0, 20000), ((1 << 22) - 5000, 10000)):
            out = np.zeros(n)
            rc = L.dfcg_normals_fetch(P.context(0), C.c_int(stream), C.c_int64(pos), C.c_int64(n),
                                      out.ctypes.data_as(C.c_void_p))
            assert rc == 0
            ref = P.SeededRng(0x737674, stream).normal(pos + n)[pos:]
            ulp = np.abs(out - ref) / np.spacing(np.abs(ref))
            assert ulp.max() <= 4, (stream, pos, ulp.max())
            assert np.mean(out == ref) > 0.5


def test_normal_stream_eviction_and_redraw():
    """With a 10-chunk device budget (DFCG_NORMALS_MAX_CHUNKS), reading far ahead evicts the
    first chunks; reading them again redraws them from their engine snapshots — the same values
    (a child process: the budget is read once per cache)."""
    code = r"""
import ctypes as C, numpy as np, sys
sys.path.insert(0, %r)
import paper_1107_0789_b200 as P
L = P.lib()
def fetch(pos, n):
    out = np.zeros(n)
    assert L.dfcg_normals_fetch(P.context(0), C.c_int(0), C.c_int64(pos), C.c_int64(n),
                                out.ctypes.data_as(C.c_void_p)) == 0
    return out
K = 1 << 22
first = fetch(0, 5000)
mid = fetch(K - 100, 300)
for c in range(1, 40):
    fetch(c * K + 7, 1000)  # walk 40 chunks: the budget forces evictions
assert np.array_equal(fetch(0, 5000), first)
assert np.array_equal(fetch(K - 100, 300), mid)
ref = P.SeededRng(0x737674, 0).normal(5000)
assert np.abs(first - ref).max() <= 4 * np.spacing(np.abs(ref)).max()
print("OK")
""" % ROOT
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       env={**os.environ, "DFCG_NORMALS_MAX_CHUNKS": "10"})
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
