set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_combine.py -x -q -k "anchor or block_failure" > gpurun_out/r02_t3.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02_t3.log
timeout 900 python tools/probe_base_full.py --iters 80 --budget 600 > gpurun_out/r02_base_full.txt 2>&1; echo "probe rc=$?"
tail -60 gpurun_out/r02_base_full.txt
