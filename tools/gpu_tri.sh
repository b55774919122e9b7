# triangulation change: full GPU suite, then c2 / c3 benches
mkdir -p gpurun_out/tri
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/tri/pytest_gpu.log 2>&1; tail -1 gpurun_out/tri/pytest_gpu.log
VARIANTS="base" WL="c2 c3" STEPS=8 bash tools/gpu_ab.sh
for f in gpurun_out/ab/c2.base.json gpurun_out/ab/c3.base.json; do python - $f <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["ms_per_step"], {a:(round(b["ms_per_step"],2),round(b["kernel_ms_per_step"],2)) for a,b in d["kernel_families"].items()})
PY
done
