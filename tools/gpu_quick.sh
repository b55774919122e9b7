# parity tests + a short C2 bench (no cpu baseline) + probes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
for c in ${PROBES:-c5 c3}; do echo "== $c"; timeout 300 python tools/probe_configs.py $c 3 2>&1 | tail -30; done > gpurun_out/probe_configs.log 2>&1
