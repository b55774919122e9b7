mkdir -p gpurun_out/ab
for w in $WL; do
for lib in $VARIANTS; do
  tag=$(echo $lib | tr '/' '_')
  if [ "$lib" = base ]; then unset RAMA_LIB; else export RAMA_LIB=$PWD/$lib; fi
  timeout 600 python bench.py --workload $w --steps ${STEPS:-8} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab/$w.$tag.json 2> gpurun_out/ab/$w.$tag.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/ab/$w.$tag.json").read().strip().splitlines()[-1])
k={x["kernel"]:x["ms_per_step"] for x in d["top_kernels"]}
print("$w %-28s ms/step %.2f sep_src %.3f mid %.3f wide %.3f primal %.6f" % ("$lib", d["ms_per_step"], k.get("k_sep_src",0), k.get("k_sep_src_mid",0), k.get("k_sep_src_wide",0), d["objective"]["primal"]))
PY
done; done
