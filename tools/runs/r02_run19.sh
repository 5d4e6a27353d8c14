set -x
mkdir -p gpurun_out
timeout 600 python tools/bench_sparse.py 20 > gpurun_out/r02_bench_sparse2.txt 2>&1; echo "rc=$?"; cat gpurun_out/r02_bench_sparse2.txt
timeout 1200 python -m pytest tests/test_gpu_apg.py tests/test_gpu_variants.py tests/test_gpu_combine.py -x -q > gpurun_out/r02_t19.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_t19.log
timeout 600 python tools/probe_c5_block.py 60 10 > gpurun_out/r02_c5blk_chunk.txt 2>&1; echo "c5blk rc=$?"; tail -11 gpurun_out/r02_c5blk_chunk.txt | head -10
