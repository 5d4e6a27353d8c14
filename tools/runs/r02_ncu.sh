# ncu evidence (round 2), one tool (ncu) in this call. Each ncu command follows the same command
# line run plain with && (the recipe in /opt/skills/guides/B200_PROFILING.md).
set -x
mkdir -p gpurun_out
export DFCG_PROFILE_ITER=30
# 1) launch list of one steady c2 iteration (block 0, iteration 30, lone: per-panel Cholesky)
python tools/prof_c2.py 31 > gpurun_out/r02_plain1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.sum \
    --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02_launches_it30.csv \
    python tools/prof_c2.py 31 > gpurun_out/r02_ncu1.log 2>&1; echo "ncu1 rc=$?"
# 2) the same iteration with the fused cooperative Cholesky (as in the packed bench)
DFCG_CHOL_FUSED=1 python tools/prof_c2.py 31 > gpurun_out/r02_plain2.log 2>&1 && \
DFCG_CHOL_FUSED=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.sum \
    --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02_launches_it30_fused.csv \
    python tools/prof_c2.py 31 > gpurun_out/r02_ncu2.log 2>&1; echo "ncu2 rc=$?"
# 3) --set full of the top kernel (gemm_kernel) in that iteration, and of chol_fused_kernel
python tools/prof_c2.py 31 > gpurun_out/r02_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:gemm_kernel -s 2 -c 3 \
    -o gpurun_out/r02_gemm python tools/prof_c2.py 31 > gpurun_out/r02_ncu3.log 2>&1; echo "ncu3 rc=$?"
DFCG_CHOL_FUSED=1 python tools/prof_c2.py 31 > gpurun_out/r02_plain4.log 2>&1 && \
DFCG_CHOL_FUSED=1 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:chol_fused -s 0 -c 2 -o gpurun_out/r02_cholfused python tools/prof_c2.py 31 > gpurun_out/r02_ncu4.log 2>&1; echo "ncu4 rc=$?"
ls -la gpurun_out
