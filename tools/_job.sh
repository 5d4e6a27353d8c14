set -x
timeout 1800 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/s4_gputest_final2.log 2>&1; tail -4 gpurun_out/s4_gputest_final2.log
timeout 900 python bench.py > gpurun_out/s4_bench_final2.json 2> gpurun_out/s4_bench_final2.err; tail -c 300 gpurun_out/s4_bench_final2.err
python -c "import __graft_entry__ as g; g.smoke()"
