# compute-sanitizer over tools/sanitize_case.py (every kernel family on small shapes):
# memcheck (out-of-bounds / misaligned / leaks of device allocations), racecheck (shared-memory
# hazards), synccheck (barrier misuse). Summaries land in gpurun_out/r02_sanitize_*.txt.
set -x
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 \
      python tools/sanitize_case.py > gpurun_out/r02_sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"
  tail -4 gpurun_out/r02_sanitize_$tool.txt
done
