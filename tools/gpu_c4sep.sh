# C4 separation: per-round stats + ncu of the first k_sep4 launch
mkdir -p gpurun_out/c4sep
RAMA_SEP_STATS=1 RAMA_ROUND_PROF=1 timeout 300 python tools/probe_configs.py c4 1 > gpurun_out/c4sep/stats.log 2>&1
grep -E "sep n=|round" gpurun_out/c4sep/stats.log | head -40
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_sep4" -s 0 -c 1 \
  -o gpurun_out/c4sep/k_sep4 -f python tools/probe_configs.py c4 1 > gpurun_out/c4sep/ncu.log 2>&1
tail -2 gpurun_out/c4sep/ncu.log
