# per-launch durations of the sort-reduce tiles in one C2 solve, and a full capture of the cleanup's contraction
mkdir -p gpurun_out/tiles
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sr_" --csv --log-file gpurun_out/tiles/launches.csv python tools/probe_configs.py c2 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_sr_tiles" -s 8 -c 1 -o gpurun_out/tiles/cl_tiles -f python tools/probe_configs.py c2 1 > gpurun_out/tiles/ncu.log 2>&1
tail -2 gpurun_out/tiles/ncu.log
