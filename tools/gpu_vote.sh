# vote pre-check + triangulation fusions: full GPU suite, A/B on c2 / c3
mkdir -p gpurun_out/vote
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/vote/pytest_gpu.log 2>&1; tail -1 gpurun_out/vote/pytest_gpu.log
VARIANTS="base abtest/noprecheck/librama_b200.so" WL="c2 c3" STEPS=8 bash tools/gpu_ab.sh
VARIANTS="base abtest/noprecheck/librama_b200.so" WL="c2" STEPS=8 bash tools/gpu_ab.sh
for f in gpurun_out/ab/c*.json; do python - $f <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k={x["kernel"]:x["ms_per_step"] for x in d["top_kernels"]}
print(sys.argv[1], d["ms_per_step"], "cl_rounds %.3f match_vote %.3f" % (k.get("k_cl_rounds",0), k.get("k_match_vote",0)), {a:round(b["kernel_ms_per_step"],2) for a,b in d["kernel_families"].items()})
PY
done
