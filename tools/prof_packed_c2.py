"""Packed c2 step for an ncu launch list: the eight c2 blocks advanced concurrently (one host
thread and stream each, as in bench.py) through iteration `skip`, then `win` more iterations.
Prints the library launch count at the start of the window (pass it to ncu -s) and the launches
per window, so `ncu -s <count> -c <launches>` captures the packed window's kernels with their
SM-time (sm__cycles_active.sum), whose shares hold under concurrency.

With a third argument "bracket" the window is bracketed by cuProfilerStart / cuProfilerStop
(ncu --profile-from-start off): the launch count at the window's start is not reproducible from
run to run since the persistent Jacobi sweeps (one launch or ~700 per SVD, chosen by how many
solves are active when the last blocks finish the skip phase). Run with DFCG_JACOBI_PERSIST=0
DFCG_JACOBI_CLUSTER=1 so the blocks that finish the window last keep the packed step's kernel
choices under ncu's serialisation."""
import ctypes
import os
import sys
from concurrent.futures import ThreadPoolExecutor

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P  # noqa: E402

skip = int(sys.argv[1]) if len(sys.argv) > 1 else 30
win = int(sys.argv[2]) if len(sys.argv) > 2 else 1
L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
groups = P.partition_columns(1, 0xDFC0000000000001, 10000, 8)
blocks = [P.extract_columns(obs, g) for g in groups]
del obs
solvers = [P.McSolver(b) for b in blocks]
pool = ThreadPoolExecutor(8)
list(pool.map(lambda s: s.step(skip), solvers))
bracket = len(sys.argv) > 3 and sys.argv[3] == "bracket"
cu = ctypes.CDLL("libcuda.so.1") if bracket else None
c0 = P.launch_count()
if cu:
    cu.cuProfilerStart()
list(pool.map(lambda s: s.step(win), solvers))
if cu:
    cu.cuProfilerStop()
print(f"window launches start {c0} count {P.launch_count() - c0}", flush=True)
for s in solvers:
    s.close()
