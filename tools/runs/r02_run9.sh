set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_baseline_scale.py tests/test_integration.py tests/test_gpu_variants.py -x -q --durations=8 > gpurun_out/r02_t9.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02_t9.log
timeout 1200 python tools/probe_c5_sweep.py 8,16,32,64 4 > gpurun_out/r02_c5_sweep.txt 2>&1; echo "c5 rc=$?"; tail -6 gpurun_out/r02_c5_sweep.txt
