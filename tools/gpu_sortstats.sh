mkdir -p gpurun_out
RAMA_SORT_STATS=1 RAMA_TRACE=${TRACE:-0} timeout 300 python tools/probe_configs.py c2 1 > gpurun_out/sortstats_c2.log 2>&1
