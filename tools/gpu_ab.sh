# A/B of library variants on a workload: VARIANTS="base abtest/x/librama_b200.so ..." WL=c2
mkdir -p gpurun_out/ab
for w in ${WL:-c2}; do
for lib in ${VARIANTS:-base}; do
  tag=$(echo $lib | tr '/' '_')
  if [ "$lib" = base ]; then unset RAMA_LIB; else export RAMA_LIB=$PWD/$lib; fi
  timeout 600 python bench.py --workload $w --steps ${STEPS:-8} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab/$w.$tag.json 2> gpurun_out/ab/$w.$tag.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/ab/$w.$tag.json").read().strip().splitlines()[-1])
k={x["kernel"]:x["ms_per_step"] for x in d["top_kernels"]}
f=d["kernel_families"]
print("$w %-32s ms/step %.2f  contract %.2f canon? sr_tiles %.3f sr_scatter %.3f sr_count %.3f primal %.6f" % ("$lib", d["ms_per_step"], f["contract"]["kernel_ms_per_step"], k.get("k_sr_tiles",0), k.get("k_sr_scatter",0), k.get("k_sr_count",0), d["objective"]["primal"]))
PY
done; done
