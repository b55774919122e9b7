# final check of HEAD as the driver runs it: GPU tests, smoke, default bench, reference arm
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/final/pytest_gpu.log 2>&1; tail -1 gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; tail -1 gpurun_out/final/smoke.log
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; tail -c 250 gpurun_out/final/bench.json
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err; tail -c 250 gpurun_out/final/bench_ref.json
