mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
( timeout 1200 $S --tool memcheck --error-exitcode 9 python tools/sanitize.py 2>&1 | tail -4
  RAMA_SEP_FALLBACK=2 RAMA_CLEANUP_POOL=64 timeout 1200 $S --tool memcheck --error-exitcode 9 python tools/sanitize.py 2>&1 | tail -3
  timeout 1800 $S --tool racecheck --error-exitcode 9 python tools/sanitize.py 2>&1 | tail -3 ) > gpurun_out/sanitize.log 2>&1; cat gpurun_out/sanitize.log

