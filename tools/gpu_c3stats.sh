mkdir -p gpurun_out/c3s
RAMA_ROUND_PROF=1 timeout 300 python tools/probe_configs.py c3 2 > gpurun_out/c3s/roundprof.log 2>&1
RAMA_HOST_STATS=2 timeout 300 python tools/probe_configs.py c3 2 > gpurun_out/c3s/hoststats.log 2>&1
RAMA_SORT_STATS=1 timeout 300 python tools/probe_configs.py c3 1 > gpurun_out/c3s/sortstats.log 2>&1
