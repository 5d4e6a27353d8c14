set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_apg.py tests/test_gpu_combine.py tests/test_gpu_variants.py tests/test_gpu_dist.py -x -q > gpurun_out/r02_t14.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_t14.log
for f in 1 0; do
  DFCG_CHOL_FUSED=$f timeout 300 python tools/probe_lone_c2.py > gpurun_out/r02_lone3_fused$f.txt 2>&1; echo "lone fused=$f rc=$?"; cat gpurun_out/r02_lone3_fused$f.txt
done
for f in 1 3; do
  DFCG_CHOL_FUSED=$f timeout 600 python bench.py --steps 20 --warmup 5 --no-extra --no-lowrank --no-cpu --no-e2e > gpurun_out/r02_bench3_fused$f.json 2>/dev/null; echo "bench fused=$f rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02_bench3_fused$f.json').read().strip().splitlines()[-1])
print('fused=$f value',d['value'],'step frac',d['roofline_step']['frac'],'launches/step',d['roofline_step']['launches_per_step'])"
done
