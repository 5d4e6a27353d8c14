set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_apg.py tests/test_gpu_variants.py -x -q > gpurun_out/r02_t7.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02_t7.log
for v in 1 0; do
  DFCG_SPMM_SLAB=$v timeout 600 python tools/probe_c5_block.py 60 10 > gpurun_out/r02_c5blk_slab$v.txt 2>&1; echo "c5 slab=$v rc=$?"
  tail -12 gpurun_out/r02_c5blk_slab$v.txt | head -11
done
