"""Per-GPU throughput with k of the eight c2 blocks sharing the GPU (k = 1, 2, 4, 8): what one
rank of an N = 8 / k GPU run executes (blocks are independent, no exchange during the solve), so
N x rate(8 / N) is the measured-per-rank prediction of the strong-scaling curve. Each k: the
first k blocks advanced concurrently through iteration 31, then 20 timed iterations each."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_0789_b200 as P  # noqa: E402

L0, obs = P.gen_mc_instance(10000, 10000, 10, 10_000_000, 0.1, 1)
groups = P.partition_columns(1, 0xDFC0000000000001, 10000, 8)
blocks = [P.extract_columns(obs, g) for g in groups]
del obs
pool = ThreadPoolExecutor(8)
for k in (1, 2, 4, 8):
    solvers = [P.McSolver(b) for b in blocks[:k]]
    list(pool.map(lambda s: s.step(31), solvers))
    t0 = time.perf_counter()
    list(pool.map(lambda s: s.step(20), solvers))
    dt = time.perf_counter() - t0
    rate = 20 * k / dt
    print(f"k = {k} blocks on the GPU: {1e3 * dt / 20:.2f} ms per step, {rate:.1f} block-it/s per GPU; "
          f"N = {8 // k} GPUs x this = {8 // k * rate:.0f} block-it/s", flush=True)
    for s in solvers:
        s.close()
