# Round-2 measurement set: bench lines (C2 with CPU baseline + e2e, C3, C4,
# C5 batch), the reference arm on C2, and the ncu launch list of one C2 bench
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2/smi.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2/bench_c2.json 2> gpurun_out/r2/bench_c2.err
for w in c3 c4 c5batch; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_$w.json 2> gpurun_out/r2/bench_$w.err
done
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/r2/bench_c2_reference.json 2> gpurun_out/r2/bench_c2_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/c2_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2/ncu_bench.log 2>&1
for f in gpurun_out/r2/bench_*.json; do echo $f; tail -c 400 $f; echo; done
