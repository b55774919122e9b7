mkdir -p gpurun_out
RAMA_CLEANUP_STATS=1 timeout 300 python tools/probe_configs.py c3 2 > gpurun_out/cleanup_c3.log 2>&1
RAMA_CLEANUP_STATS=1 timeout 300 python tools/probe_configs.py c2 3 >> gpurun_out/cleanup_c3.log 2>&1
