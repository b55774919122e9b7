# state check: gpu tests, smoke, short C2 bench
mkdir -p gpurun_out/chk
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/chk/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/chk/bench_c2.json 2> gpurun_out/chk/bench_c2.err
tail -3 gpurun_out/chk/pytest_gpu.log; tail -c 600 gpurun_out/chk/bench_c2.json
