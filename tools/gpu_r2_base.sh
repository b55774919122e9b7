# round-2 baseline: bench lines for every workload + per-phase round timing
mkdir -p gpurun_out/r2base
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2base/smi.txt
for w in c2 c3 c4 c5batch; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2base/bench_$w.json 2> gpurun_out/r2base/bench_$w.err
done
RAMA_ROUND_PROF=1 RAMA_HOST_STATS=1 timeout 300 python tools/probe_configs.py c2 2 > gpurun_out/r2base/prof_c2.log 2>&1
RAMA_ROUND_PROF=1 RAMA_HOST_STATS=1 timeout 300 python tools/probe_configs.py c4 1 > gpurun_out/r2base/prof_c4.log 2>&1
