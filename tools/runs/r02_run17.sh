set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_apg.py tests/test_gpu_variants.py -x -q > gpurun_out/r02_t17.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_t17.log
timeout 300 python tools/probe_lone_c2.py > gpurun_out/r02_lone17.txt 2>&1; echo "lone rc=$?"; head -12 gpurun_out/r02_lone17.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-extra --no-lowrank --no-cpu --no-e2e > gpurun_out/r02_bench17.json 2>/dev/null; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/r02_bench17.json').read().strip().splitlines()[-1])
print('value',d['value'],'step frac',d['roofline_step']['frac'],'launches/step',d['roofline_step']['launches_per_step'])"
CHOL_BENCH_P=16,32 timeout 900 python tools/bench_cholesky.py > gpurun_out/r02_bench_cholesky17.txt 2>&1; cat gpurun_out/r02_bench_cholesky17.txt
