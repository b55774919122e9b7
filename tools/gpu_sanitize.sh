mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
( timeout 1200 $S --tool memcheck --error-exitcode 9 python tools/sanitize.py 2>&1 | tail -4
  RAMA_SEP_FALLBACK=2 RAMA_CLEANUP_POOL=64 timeout 1200 $S --tool memcheck --error-exitcode 9 python tools/sanitize.py 2>&1 | tail -3
  timeout 1800 $S --tool racecheck --error-exitcode 9 python tools/sanitize.py 2>&1 | tail -3 ) > gpurun_out/sanitize.log 2>&1
for c in c4 c5; do RAMA_HOST_STATS=1 timeout 600 python tools/probe_configs.py $c 2 > gpurun_out/probe_$c.log 2>&1; done
