set -x
mkdir -p gpurun_out
timeout 1500 python tools/probe_c5_sweep.py 8,16,32,64 4 > gpurun_out/r02_c5_sweep2.txt 2>&1; echo "c5 rc=$?"; tail -5 gpurun_out/r02_c5_sweep2.txt
timeout 2400 python tools/probe_c4_full.py 64 16 > gpurun_out/r02_c4_full.txt 2>&1; echo "c4 rc=$?"; tail -3 gpurun_out/r02_c4_full.txt
bash tools/runs/r02_sanitize.sh
