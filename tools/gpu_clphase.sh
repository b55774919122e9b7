mkdir -p gpurun_out
RAMA_CLEANUP_STATS=3 timeout 300 python tools/probe_configs.py c3 1 > gpurun_out/clphase_c3.log 2>&1
RAMA_CLEANUP_STATS=3 timeout 300 python tools/probe_configs.py c2 1 > gpurun_out/clphase_c2.log 2>&1
