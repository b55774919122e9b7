mkdir -p gpurun_out
RAMA_HOST_STATS=1 RAMA_CLEANUP_STATS=1 timeout 600 python tools/probe_configs.py c4 2 > gpurun_out/c4.log 2>&1
