set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_baseline_scale.py -x -q -k "c1 or combine" 2>&1 | tail -15
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench1.json 2> gpurun_out/r02_bench1.err
tail -c 3000 gpurun_out/r02_bench1.json
