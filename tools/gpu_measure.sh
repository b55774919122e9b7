# Full measurement set: bench lines (C2 with CPU baseline + e2e, C3, C4, C5 batch),
# the reference arm on C2, the ncu launch list of a C2 bench, ncu --set full captures
O=gpurun_out/meas; mkdir -p $O/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
for w in c3 c4 c5batch; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > $O/bench_c2_reference.json 2> $O/bench_c2_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_bench.log 2>&1
cap() {  # label regex skip
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 1 \
    -o $O/ncu/r02_c2_$1 -f python tools/probe_configs.py c2 1 > $O/ncu/$1.log 2>&1
  tail -1 $O/ncu/$1.log
}
cap k_sep_src "^k_sep_src" 0
cap k_cl_rounds "^k_cl_rounds" 0
cap k_mp_edge "^k_mp_edge" 0
cap k_mp_triplet "^k_mp_triplet" 0
cap k_sr_count "^k_sr_count" 1
cap k_sr_scatter "^k_sr_scatter" 1
cap k_sr_tiles "^k_sr_tiles" 1
cap k_sr_tiles_cleanup "^k_sr_tiles" 8
cap k_match_vote "^k_match_vote" 0
cap k_reparam "^k_reparam" 0
cap k_tri_handles "^k_tri_handles" 0
cap k_slot_count "^k_slot_count" 0
for f in $O/bench_*.json; do echo $f; tail -c 300 $f; echo; done
