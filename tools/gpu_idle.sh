# where the C2 step idles: host sync call chains and the kernel timeline gaps
mkdir -p gpurun_out/idle
RAMA_HOST_STATS=2 timeout 300 python tools/probe_configs.py c2 2 > gpurun_out/idle/hoststats2.log 2>&1
timeout 300 python tools/timeline.py c2 gpurun_out/idle/timeline_c2.json > gpurun_out/idle/timeline.log 2>&1
tail -5 gpurun_out/idle/timeline.log
