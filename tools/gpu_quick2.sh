# quick loop: parity subset (or all with FULL=1) + C2 bench (+ optional extra workloads)
mkdir -p gpurun_out/q
if [ -n "$FULL" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/q/pytest.log 2>&1
else
  timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "${TESTS:-canonicalize or contract or ops_oracle or c2_full or c5_instance or small_pd or grid_pd}" > gpurun_out/q/pytest.log 2>&1
fi
tail -5 gpurun_out/q/pytest.log
for w in ${WL:-c2}; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q/bench_$w.json 2> gpurun_out/q/bench_$w.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/q/bench_$w.json").read().strip().splitlines()[-1])
print("$w ms/step %.2f launches/step %.0f primal %.6f lb %.6f" % (d["ms_per_step"], d["gpu_launches"]/d["steps"], d["objective"]["primal"], d["objective"]["lower_bound"]))
print(" fam", {k:(round(v["ms_per_step"],2), round(v["kernel_ms_per_step"],2)) for k,v in d["kernel_families"].items()})
print(" top", [(k["kernel"], round(k["ms_per_step"],3), k["launches_per_step"]) for k in d["top_kernels"][:14]])
PY
done
