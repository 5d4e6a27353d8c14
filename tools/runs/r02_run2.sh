set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r02_gputest2.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r02_gputest2.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r02_bench2.json
