mkdir -p gpurun_out
RAMA_CLEANUP_STATS=2 timeout 300 python tools/probe_configs.py c2 2 > gpurun_out/cltrace_c2.log 2>&1
RAMA_CLEANUP_STATS=2 timeout 300 python tools/probe_configs.py c3 2 > gpurun_out/cltrace_c3.log 2>&1
