mkdir -p gpurun_out
K=${KREGEX:-k_sep_src}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-0} -c ${COUNT:-1} -o gpurun_out/prof_$TAG python tools/probe_configs.py c2 1 > gpurun_out/ncu_$TAG.log 2>&1
