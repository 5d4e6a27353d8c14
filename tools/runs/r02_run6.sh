set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --no-extra --no-lowrank --no-cpu > gpurun_out/r02_bench6.json 2> gpurun_out/r02_bench6.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/r02_bench6.json').read().strip().splitlines()[-1])
print('value',d['value'],'e2e',d['e2e']['value'],d['e2e']['divide_ms'],'step frac',d['roofline_step']['frac'])"
