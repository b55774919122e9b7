# sort-reduce variants: parity tests on the in-tree build, then A/B on c2 / c3
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_ops.py -m gpu -q -x --timeout 600 > gpurun_out/ab/pytest_ops.log 2>&1; tail -1 gpurun_out/ab/pytest_ops.log
VARIANTS="base abtest/quad/librama_b200.so abtest/blocklb/librama_b200.so abtest/short128/librama_b200.so" WL="c2 c3" STEPS=6 bash tools/gpu_ab.sh
