set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_solver_api.py -x -q > gpurun_out/r02_t4.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/r02_t4.log
