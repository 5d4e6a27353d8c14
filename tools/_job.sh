set -x
DFCG_JACOBI_P2P=0 timeout 300 python tools/probe_lone_c2.py > gpurun_out/s4_lone_p2p0.txt 2>&1; cat gpurun_out/s4_lone_p2p0.txt
DFCG_JACOBI_P2P=1 timeout 300 python tools/probe_lone_c2.py > gpurun_out/s4_lone_p2p1.txt 2>&1; cat gpurun_out/s4_lone_p2p1.txt
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_apg.py tests/test_gpu_baseline_scale.py tests/test_gpu_combine.py -q -x --durations=3 > gpurun_out/s4_gputest_p2p.log 2>&1; tail -8 gpurun_out/s4_gputest_p2p.log
timeout 600 python bench.py --no-cpu --no-lowrank --steps 20 --warmup 5 > gpurun_out/s4_bench_p2p.json 2> gpurun_out/s4_bench_p2p.err
python - <<P
import json
d=json.loads(open('gpurun_out/s4_bench_p2p.json').read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['dfc_proj_solve_s'],2), round(d['base_apg']['value'],3), round(d['nys_c2']['solve_s'],2), round(d['rmf_c3']['solve_s'],2))
P
