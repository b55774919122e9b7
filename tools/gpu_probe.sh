mkdir -p gpurun_out
for c in c5 c3 c4; do
  echo "== $c"; timeout 400 python tools/probe_configs.py $c 3 2>&1 | tail -40
done > gpurun_out/probe_configs.log 2>&1
