set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -x -q -k "JACOBI or SPMM_CHUNK" > gpurun_out/r02_t20.log 2>&1; echo "variants rc=$?"; tail -3 gpurun_out/r02_t20.log
DFCG_JACOBI_PERSIST=0 timeout 300 python tools/probe_lone_c2.py > gpurun_out/r02_lone20_p0.txt 2>&1; echo "lone p0 rc=$?"; cat gpurun_out/r02_lone20_p0.txt
timeout 300 python tools/probe_lone_c2.py > gpurun_out/r02_lone20_p2.txt 2>&1; echo "lone p2 rc=$?"; cat gpurun_out/r02_lone20_p2.txt
DFCG_JACOBI_CLUSTER=1 timeout 300 python tools/probe_lone_c2.py > gpurun_out/r02_lone20_p2c1.txt 2>&1; echo "lone p2 c1 rc=$?"; cat gpurun_out/r02_lone20_p2c1.txt
DFCG_JACOBI_CLUSTER=4 timeout 300 python tools/probe_lone_c2.py > gpurun_out/r02_lone20_p2c4.txt 2>&1; echo "lone p2 c4 rc=$?"; cat gpurun_out/r02_lone20_p2c4.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-extra --no-lowrank --no-cpu --no-e2e > gpurun_out/r02_bench20_p2.json 2>/dev/null; echo "bench rc=$?"
DFCG_JACOBI_PERSIST=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-extra --no-lowrank --no-cpu --no-e2e > gpurun_out/r02_bench20_p1.json 2>/dev/null; echo "bench p1 rc=$?"
for f in p2 p1; do python -c "
import json;d=json.loads(open('gpurun_out/r02_bench20_$f.json').read().strip().splitlines()[-1])
print('$f value',d['value'],'step frac',d['roofline_step']['frac'],'launches/step',d['roofline_step']['launches_per_step'])"; done
timeout 600 python tools/probe_nys.py > gpurun_out/r02_nys20.txt 2>&1; echo "nys rc=$?"; cat gpurun_out/r02_nys20.txt
