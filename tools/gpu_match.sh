# cooperative matching: GPU suite, A/B against one launch pair per round
mkdir -p gpurun_out/match
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/match/pytest_gpu.log 2>&1; tail -1 gpurun_out/match/pytest_gpu.log
VARIANTS="base" WL="c2 c3" STEPS=8 bash tools/gpu_ab.sh
RAMA_MATCH_LAUNCHES=1 VARIANTS="base" WL="c2 c3" STEPS=8 bash tools/gpu_ab.sh
