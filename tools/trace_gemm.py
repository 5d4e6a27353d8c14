"""GEMM shapes and per-call times of one steady-state c2 APG iteration (block 0, iteration N+1,
run alone): DFCG_TRACE_GEMM=1 python tools/trace_gemm.py [N]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
groups = P.partition_columns(1, 0xDFC0000000000001, 10000, 8)
s = P.McSolver(P.extract_columns(obs, groups[0]), P.ApgConfig())
s.step(n)
P.prof_enable(True)
s.step(1)
P.prof_enable(False)
