set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:jacobi_sweeps --launch-skip 30 -c 1 -f -o gpurun_out/r02_jsweeps python tools/probe_lone_c2.py > gpurun_out/r02_ncu21.log 2>&1; echo "ncu rc=$?"; tail -5 gpurun_out/r02_ncu21.log
