# small-tree forest path: forest tests, full gpu suite, A/B vs the Euler-tour path, round profile
mkdir -p gpurun_out/forest
timeout 900 python -m pytest tests/test_gpu_ops.py -m gpu -q -x --timeout 600 -k "forest or selection" > gpurun_out/forest/pytest_forest.log 2>&1; tail -1 gpurun_out/forest/pytest_forest.log
RAMA_FOREST_TOUR=1 timeout 900 python -m pytest tests/test_gpu_ops.py -m gpu -q -x --timeout 600 -k "forest" > gpurun_out/forest/pytest_forest_tour.log 2>&1; tail -1 gpurun_out/forest/pytest_forest_tour.log
RAMA_ROUND_PROF=1 timeout 300 python tools/probe_configs.py c2 2 > gpurun_out/forest/roundprof_c2.log 2>&1
VARIANTS="base" WL="c2 c3" STEPS=8 bash tools/gpu_ab.sh
RAMA_FOREST_TOUR=1 VARIANTS="base" WL="c2 c3" STEPS=8 bash tools/gpu_ab.sh
RAMA_CLEANUP_STATS=2 timeout 300 python tools/probe_configs.py c3 1 > gpurun_out/forest/cltrace_c3.log 2>&1
RAMA_CLEANUP_STATS=2 timeout 300 python tools/probe_configs.py c2 1 > gpurun_out/forest/cltrace_c2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/forest/pytest_gpu.log 2>&1; tail -1 gpurun_out/forest/pytest_gpu.log
