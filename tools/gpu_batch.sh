# batch tests + c5batch bench at 1 / 2 union groups
mkdir -p gpurun_out/b
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "batch or c5" > gpurun_out/b/pytest.log 2>&1
tail -3 gpurun_out/b/pytest.log
for w in ${NGRP:-1 2}; do
  RAMA_BATCH_WORKERS=$w timeout 600 python bench.py --workload c5batch --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b/bench_$w.json 2> gpurun_out/b/bench_$w.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/b/bench_$w.json").read().strip().splitlines()[-1])
print("groups $w ms/step %.2f launches/step %.0f" % (d["ms_per_step"], d["gpu_launches"]/d["steps"]))
print(" fam", {k:(round(v["ms_per_step"],2), round(v["kernel_ms_per_step"],2)) for k,v in d["kernel_families"].items()})
print(" top", [(k["kernel"], round(k["ms_per_step"],3), k["launches_per_step"]) for k in d["top_kernels"][:12]])
PY
done
