# ncu --set full of one launch of kernel $K (regex), skipping $SKIP launches, on probe_configs $CFG
mkdir -p gpurun_out/ncu
K=${K:-k_sr_tiles}; SKIP=${SKIP:-1}; CFG=${CFG:-c2}; TAG=${TAG:-$K}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $SKIP -c ${COUNT:-1} \
  -o gpurun_out/ncu/$TAG -f python tools/probe_configs.py $CFG 1 > gpurun_out/ncu/$TAG.log 2>&1
tail -3 gpurun_out/ncu/$TAG.log
