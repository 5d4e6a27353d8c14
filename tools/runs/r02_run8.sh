set -x
mkdir -p gpurun_out
timeout 600 python tools/bench_sparse.py 20 > gpurun_out/r02_bench_sparse.txt 2>&1; echo "rc=$?"; cat gpurun_out/r02_bench_sparse.txt | tail -5
