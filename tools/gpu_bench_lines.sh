# bench lines (C2 with CPU baseline + e2e, C3, C4, C5 batch) and the C2 ncu launch list
O=gpurun_out/meas2; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
for w in c3 c4 c5batch; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"DeviceRadixSortOnesweep" -s 40 -c 1 \
  -o $O/r02_c2_quotient_onesweep -f python tools/probe_configs.py c2 1 > $O/ncu_onesweep.log 2>&1
for f in $O/bench_*.json; do echo $f; tail -c 300 $f; echo; done
