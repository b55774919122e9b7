# cooperative Boruvka: GPU suite, A/B against one launch set per iteration
mkdir -p gpurun_out/bv
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/bv/pytest_gpu.log 2>&1; tail -1 gpurun_out/bv/pytest_gpu.log
RAMA_ROUND_PROF=1 timeout 300 python tools/probe_configs.py c2 2 2>&1 | grep forest | tail -2
VARIANTS="base" WL="c2 c3" STEPS=8 bash tools/gpu_ab.sh
RAMA_BORUVKA_LAUNCHES=1 VARIANTS="base" WL="c2 c3" STEPS=8 bash tools/gpu_ab.sh
