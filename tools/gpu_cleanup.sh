mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
RAMA_CLEANUP_STATS=1 timeout 300 python tools/probe_configs.py c3 2 > gpurun_out/cleanup_c3.log 2>&1
RAMA_CLEANUP_STATS=1 timeout 300 python tools/probe_configs.py c2 2 >> gpurun_out/cleanup_c3.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
bash tools/gpu_cltrace.sh
