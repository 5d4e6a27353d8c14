"""CPU-only checks of the product's host side: the C-ABI library loads and exports every
symbol include/*.h declares, its host RNG / sampling / generators reproduce the reference's
golden vectors and the oracle bit for bit, and compute calls refuse to run without a GPU."""
import json
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1107_0789_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_pins.json")))


def declared_functions():
    names = []
    for h in ("dfcg.h", "dfcg_host.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^\s*(?:int|void|const char\*|int64_t)\s+\**(dfcg_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    L = P.lib()
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name


def test_host_rng_golden():  # P/tests/test_rng.cpp:11-48
    r = P.SeededRng(42, 0)
    assert [int(x) for x in r.u64(4)] == [int(v, 16) for v in GOLD["rng_raw_42_0"]["values"]]
    assert list(r.uniform(3)) == GOLD["rng_uniform_42_0"]["values"]
    assert list(r.normal(2)) == GOLD["rng_normal_42_0"]["values"]
    assert [int(x) for x in r.index(5, 10)] == GOLD["rng_index10_42_0"]["values"]
    assert int(P.SeededRng(42, 1).u64(1)[0]) == int(GOLD["rng_raw_42_1"]["values"][0], 16)
    with pytest.raises(ValueError):
        P.SeededRng(5, 0).index(1, 0)


def test_host_normal_stream_matches_oracle():  # the SVT draws from SeededRng(0x737674, 0|1)
    for stream in (0, 1):
        assert np.array_equal(P.SeededRng(0x737674, stream).normal(5000), O.rng_normal(0x737674, stream, 5000))


def test_bulk_mt19937_64_matches_engine():
    """The device normal cache draws its raw words with the vectorised bulk mt19937_64
    (rng.hpp Mt64): the same words as the reference's SeededRng engine, across twist
    boundaries, for both SVT streams and another seed."""
    import ctypes as C

    L = P.lib()
    L.dfcg_rng_u64.restype = None
    L.dfcg_rng_u64_bulk.restype = None
    for seed, stream, n in ((0x737674, 0, 312 * 7 + 5), (0x737674, 1, 100_000), (42, 3, 1)):
        a = np.zeros(n, np.uint64)
        b = np.zeros(n, np.uint64)
        L.dfcg_rng_u64(C.c_uint64(seed), C.c_uint64(stream), C.c_int64(n), a.ctypes.data_as(C.c_void_p))
        L.dfcg_rng_u64_bulk(C.c_uint64(seed), C.c_uint64(stream), C.c_int64(n), b.ctypes.data_as(C.c_void_p))
        assert np.array_equal(a, b), (seed, stream, n)
    assert int(P.SeededRng(42, 3).u64(1)[0]) == int(b[0])


def test_generators_match_oracle_bitwise():
    L0p, obp = P.gen_mc_instance(60, 50, 3, 900, 0.1, 5)
    L0o, obo = O.gen_mc_instance(60, 50, 3, 900, 0.1, 5, 0)
    assert np.array_equal(L0p.left, L0o.left) and np.array_equal(L0p.right, L0o.right)
    for a, b in ((obp.rows, obo.rows), (obp.cols, obo.cols), (obp.vals, obo.vals)):
        assert np.array_equal(a, b)
    Lp, Sp, Mp = P.gen_rmf_instance(30, 40, 2, 100, 0.05, 3)
    Lo, So, Mo = O.gen_rmf_instance(30, 40, 2, 100, 0.05, 3, 0)
    assert np.array_equal(Mp, Mo) and all(np.array_equal(a, b) for a, b in zip(Sp, So))
    Lp, Sp, Mp = P.gen_rmf_instance(30, 40, 2, 100, 0.01, 4, lo=-10.0, hi=10.0)
    Lo, So, Mo = O.gen_rmf_instance(30, 40, 2, 100, 0.01, 4, 0, -10.0, 10.0)
    assert np.array_equal(Mp, Mo)


def test_generator_validation():
    with pytest.raises(ValueError):
        P.gen_mc_instance(4, 4, 1, 0, 0.1, 1)
    with pytest.raises(ValueError):
        P.gen_mc_instance(4, 4, 1, 17, 0.1, 1)
    with pytest.raises(ValueError):
        P.gen_mc_instance(4, 4, 5, 4, 0.1, 1)


def test_sampling_matches_oracle():
    for n, t in ((100, 7), (17, 17), (1000, 64)):
        gp = P.partition_columns(3, 0xDFC0000000000001, n, t)
        go = O.partition_columns(3, 0xDFC0000000000001, n, t)
        assert all(np.array_equal(a, b) for a, b in zip(gp, go))
    assert np.array_equal(P.sample_without_replacement(9, 2, 50, 13), O.sample_without_replacement(9, 2, 50, 13))
    with pytest.raises(ValueError):
        P.partition_columns(1, 0, 5, 6)


def test_extract_matches_oracle():
    L0, obs = P.gen_mc_instance(40, 30, 2, 500, 0.1, 2)
    oo = O.Observed(obs.m, obs.n, obs.rows, obs.cols, obs.vals)
    idx = np.array([3, 7, 8, 20, 29])
    a, b = P.extract_columns(obs, idx), O.extract_columns(oo, idx)
    assert (a.m, a.n) == (b.m, b.n)
    assert np.array_equal(a.rows, b.rows) and np.array_equal(a.cols, b.cols) and np.array_equal(a.vals, b.vals)
    a, b = P.extract_rows(obs, idx), O.extract_rows(oo, idx)
    assert np.array_equal(a.rows, b.rows) and np.array_equal(a.cols, b.cols) and np.array_equal(a.vals, b.vals)
    with pytest.raises(ValueError):
        P.extract_columns(obs, [1, 1])
    with pytest.raises(IndexError):
        P.extract_rows(obs, [40])


def test_median_rank():  # P/tests/test_dfc.cpp:43-49
    assert P.median_rank([2, 3, 5]) == 3
    assert P.median_rank([2, 4]) == 2
    assert P.median_rank([0, 0, 0]) == 1
    assert P.median_rank([7]) == 7
    with pytest.raises(ValueError):
        P.median_rank([])


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_compute_fails_loudly_without_gpu():
    L0, obs = P.gen_mc_instance(20, 20, 2, 200, 0.1, 1)
    with pytest.raises(P.DfcError):
        P.apg_mc(obs)


def test_recsys_generator_c4_standin():
    """BASELINE c4 stand-in (no reference generator; parity of the generator itself is unpinned):
    deterministic, column-major sorted unique cells, ratings in {1..5} with the 3.6 offset, Zipf
    skew (the most popular row far above the mean), and a column-subset block that is the same as
    the cells of the full instance restricted to those columns in distribution (checked on the
    density and the rating mean)."""
    m, n, r = 400, 3000, 5
    full = P.gen_recsys_instance(m, n, r, 0.02, 7)
    again = P.gen_recsys_instance(m, n, r, 0.02, 7)
    assert np.array_equal(full.rows, again.rows) and np.array_equal(full.vals, again.vals)
    key = full.cols * m + full.rows
    assert np.all(np.diff(key) > 0)  # sorted column-major, no duplicates
    assert set(np.unique(full.vals)) <= {1.0, 2.0, 3.0, 4.0, 5.0}
    assert 3.2 < full.vals.mean() < 4.0
    assert 0.5 * 0.02 * m * n < full.count <= 0.02 * m * n * 1.001
    rc = np.bincount(full.rows, minlength=m)
    assert rc.max() > 5 * rc.mean()
    groups = P.partition_columns(7, 0xDFC0000000000001, n, 8)
    blk = P.gen_recsys_instance(m, n, r, 0.02, 7, cols=groups[0])
    assert blk.n == len(groups[0]) and blk.cols.max() < blk.n
    assert 3.2 < blk.vals.mean() < 4.0


def test_experiment_csv_schema():
    """The experiment harness writes the reference's CSV (P/include/dfc/bench.hpp:339-351):
    header, %.12g RMSE, %.6g timings; summary rows follow the per-seed rows."""
    import io

    from paper_1107_0789_b200.experiment import ExperimentSpec, ResultRow, _validate, config_echo, write_csv

    buf = io.StringIO()
    write_csv(buf, [ResultRow("proj", 3, 0.123456789012345, 1.0, 2345.678901, 0.5, 2347.2, 12),
                    ResultRow("proj_mean", 1, 0.1, 0, 0, 0, 0, 12)])
    lines = buf.getvalue().splitlines()
    assert lines[0] == "method,seed,rmse,ms_divide,ms_factor,ms_combine,ms_total,rank"
    assert lines[1] == "proj,3,0.123456789012,1,2345.68,0.5,2347.2,12"
    spec = ExperimentSpec(m=10, n=10, r=2, s=50, sigma=0.1, methods=["proj", "nys"], seeds=[1])
    assert config_echo(spec).startswith("task=mc;m=10;n=10;r=2;s=50;sigma=0.1;t=4")
    for bad in (dict(seeds=[]), dict(methods=["nope"]), dict(t=0), dict(l_frac=0.0)):
        with pytest.raises(ValueError):
            _validate(ExperimentSpec(**{**spec.__dict__, **bad}))


@pytest.mark.parametrize("n,l", [(1_000_003, 50_000), (5000, 5000), (777, 1), (200_000, 150_000)])
def test_sample_without_replacement_sparse_path_identical(n, l, monkeypatch):
    """The hash-map partial Fisher-Yates (large populations: BASELINE c5 draws 8e7 of 1.6e9
    cells) returns exactly the dense permutation's sample (P/include/dfc/sampling.hpp:15-26)."""
    monkeypatch.setenv("DFCG_SWR_SPARSE", "0")
    dense = P.sample_without_replacement(11, 3, n, l)
    monkeypatch.setenv("DFCG_SWR_SPARSE", "1")
    sparse = P.sample_without_replacement(11, 3, n, l)
    assert np.array_equal(dense, sparse)
    assert np.array_equal(dense, O.sample_without_replacement(11, 3, n, l))


def test_dstep_parallel_extraction_matches_oracle():
    """libdfcg's D step (extract_subproblems: every column group of a partition plan plus a row
    sample in one parallel stable pass) equals the oracle's extract_columns / extract_rows
    (P/include/dfc/sampling.hpp:83-113), entry for entry and in order, at several thread counts."""
    import os

    L0, obs = P.gen_mc_instance(300, 260, 3, 30000, 0.1, 6)
    oo = O.Observed(obs.m, obs.n, obs.rows, obs.cols, obs.vals)
    groups = P.partition_columns(6, 0xDFC0000000000001, obs.n, 7)
    rows = np.sort(P.sample_without_replacement(6, 0xDFC0000000000002, obs.m, 70))
    for threads in ("1", "3", "8"):
        os.environ["DFCG_DSTEP_THREADS"] = threads  # read once per process: first value wins
        subs = P.extract_subproblems(obs, groups, rows)
        assert len(subs) == 8
        for g, s in enumerate(subs[:-1]):
            ref = O.extract_columns(oo, groups[g])
            assert (s.m, s.n) == (ref.m, ref.n)
            assert np.array_equal(s.rows, ref.rows) and np.array_equal(s.cols, ref.cols)
            assert np.array_equal(s.vals, ref.vals)
        ref = O.extract_rows(oo, rows)
        assert np.array_equal(subs[-1].rows, ref.rows) and np.array_equal(subs[-1].cols, ref.cols)
        assert np.array_equal(subs[-1].vals, ref.vals)
    assert sum(s.count for s in subs[:-1]) == obs.count
    with pytest.raises(ValueError):
        P.extract_subproblems(obs, [[0, 1], [1, 2]])  # overlapping groups
    with pytest.raises(IndexError):
        P.extract_subproblems(obs, [[0, obs.n]])
