# e2e staging tuning: memcpy threads / chunk size
for cfg in "6 4" "10 4" "14 4" "10 8" "6 8"; do
  set -- $cfg
  RAMA_STAGE_THREADS=$1 RAMA_STAGE_CHUNK_MB=$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/stage_$1_$2.json 2>/dev/null
  python - $1 $2 <<'PY'
import json,sys
d=json.loads(open("gpurun_out/stage_%s_%s.json"%(sys.argv[1],sys.argv[2])).read().strip().splitlines()[-1])
print("threads", sys.argv[1], "chunk MB", sys.argv[2], "e2e ms", round(d["e2e"]["ms_per_step"],2), "device ms", round(d["ms_per_step"],2))
PY
done
nproc
