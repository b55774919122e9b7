# short C2 measurement: sort stats + 3 reps of probe + short bench
mkdir -p gpurun_out
RAMA_SORT_STATS=1 timeout 300 python tools/probe_configs.py c2 3 > gpurun_out/quick_c2.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
