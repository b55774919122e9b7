# C4 parity tests + separation tests + C4 probe (scaled and full, exact vs capped)
mkdir -p gpurun_out/c4
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "c4 or separation or hub" > gpurun_out/c4/pytest.log 2>&1
tail -5 gpurun_out/c4/pytest.log
RAMA_TRACE=0 timeout 900 python tools/c4_probe.py ${FULL:+full} > gpurun_out/c4/probe.log 2> gpurun_out/c4/probe.err
cat gpurun_out/c4/probe.log
