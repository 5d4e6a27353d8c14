set -x
mkdir -p gpurun_out
timeout 1200 python tools/bench_cholesky.py > gpurun_out/r02_bench_cholesky.txt 2>&1; echo "cholbench rc=$?"; cat gpurun_out/r02_bench_cholesky.txt
python tools/prof_packed_c2.py 30 1 > gpurun_out/r02_packed_plain.log 2>&1; echo "plain rc=$?"; cat gpurun_out/r02_packed_plain.log
S=$(grep -o "start [0-9]*" gpurun_out/r02_packed_plain.log | awk '{print $2}')
C=$(grep -o "count [0-9]*" gpurun_out/r02_packed_plain.log | awk '{print $2}')
python tools/prof_packed_c2.py 30 1 > gpurun_out/r02_packed_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s $S -c $C --csv --log-file gpurun_out/r02_launches_packed_it31.csv python tools/prof_packed_c2.py 30 1 > gpurun_out/r02_ncu_packed.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out | tail -5
