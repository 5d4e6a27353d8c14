set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r02_gputest15.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02_gputest15.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke15.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/r02_smoke15.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench15.json 2> gpurun_out/r02_bench15.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/r02_bench15.json').read().strip().splitlines()[-1])
print('value',d['value'],'e2e',d['e2e']['value'],d['e2e']['dfc_proj_solve_s'],'divide',d['e2e']['divide_ms'],'step frac',d['roofline_step']['frac'],'roof',d['roofline']['kernel'],d['roofline']['frac'],'base',d['base_apg']['value'],'nys',d['nys_c2']['solve_s'],'c3',d['rmf_c3']['solve_s'],'cpu',d['cpu_baseline']['value'],'clk',d['clocks'])"
