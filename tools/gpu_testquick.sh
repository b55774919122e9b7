mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
bash tools/gpu_sepstats.sh
bash tools/gpu_quickc2.sh
