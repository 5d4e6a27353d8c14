set -x
DFCG_BENCH_LDX=36 timeout 600 python tools/bench_sparse.py 20 > gpurun_out/s4_sparse_wide36.txt 2>&1
DFCG_BENCH_LDX=48 timeout 600 python tools/bench_sparse.py 20 > gpurun_out/s4_sparse_wide48.txt 2>&1
python - <<'P'
import json
for f in ('gpurun_out/s4_sparse_wide36.txt','gpurun_out/s4_sparse_wide48.txt'):
    for line in open(f):
        try: d=json.loads(line)
        except Exception: print(line[:300]); continue
        print(f, d['case'], {k:{m:v['us'] for m,v in d[k].items()} for k in ('spmm','spmm_t')})
P
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sddmm -c 2 -o gpurun_out/s4_sddmm_c5 -f python tools/prof_sparse.py > gpurun_out/s4_ncu_sddmm.log 2>&1
tail -2 gpurun_out/s4_ncu_sddmm.log
for run in 8 16; do DFCG_CHOLQR_WARM_RUN=$run timeout 600 python bench.py --no-cpu --no-lowrank --no-extra > gpurun_out/s4_bench_run$run.json 2> gpurun_out/s4_bench_run$run.err; done
python - <<'P'
import json
for r in (8,16):
    d=json.loads(open(f'gpurun_out/s4_bench_run{r}.json').read().strip().splitlines()[-1])
    print(r, d['value'], d['e2e']['value'], d['e2e']['dfc_proj_solve_s'])
P
