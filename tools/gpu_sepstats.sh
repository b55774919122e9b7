mkdir -p gpurun_out
RAMA_SEP_STATS=1 timeout 300 python tools/probe_configs.py c2 1 > gpurun_out/sepstats.log 2>&1
RAMA_SEP_STATS=1 timeout 300 python tools/probe_configs.py c3 1 >> gpurun_out/sepstats.log 2>&1
