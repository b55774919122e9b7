# full measurement set for profiles/: tests, smoke, bench (both arms), c5batch, launch list, ncu captures
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 600 python bench.py --workload c5batch --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu.log 2>&1
for k in k_sep_src k_cl_rounds k_mp_edge k_mp_triplet k_bucket_scatter k_rank_rows; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k" -c 1 -o gpurun_out/prof_$k python tools/probe_configs.py c2 1 > gpurun_out/ncu_$k.log 2>&1
done
