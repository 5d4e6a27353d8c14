set -x
mkdir -p gpurun_out
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench5.json 2> gpurun_out/r02_bench5.err; echo "bench rc=$?"
tail -c 2500 gpurun_out/r02_bench5.json
tail -5 gpurun_out/r02_bench5.err
