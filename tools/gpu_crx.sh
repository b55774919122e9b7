# radix contraction: GPU suite, A/B default (quotient only) / never / always
mkdir -p gpurun_out/crx
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/crx/pytest_gpu.log 2>&1; tail -1 gpurun_out/crx/pytest_gpu.log
RAMA_CONTRACT_RADIX=1 timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_solve.py -m gpu -q -x --timeout 900 > gpurun_out/crx/pytest_forced.log 2>&1; tail -1 gpurun_out/crx/pytest_forced.log
VARIANTS="base" WL="c2 c3" STEPS=8 bash tools/gpu_ab.sh
RAMA_CONTRACT_RADIX=0 VARIANTS="base" WL="c2 c3" STEPS=8 bash tools/gpu_ab.sh
RAMA_CONTRACT_RADIX=1 VARIANTS="base" WL="c2 c3" STEPS=8 bash tools/gpu_ab.sh
