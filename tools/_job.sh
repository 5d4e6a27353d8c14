set -x
timeout 1500 python tools/probe_c5_sweep.py > gpurun_out/s4_c5_sweep.txt 2>&1; grep -v '"config"' gpurun_out/s4_c5_sweep.txt | cut -c1-420
timeout 1200 python tools/probe_c4_full.py > gpurun_out/s4_c4_full.txt 2>&1; tail -2 gpurun_out/s4_c4_full.txt | cut -c1-600
