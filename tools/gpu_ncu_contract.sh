# ncu --set full of the round-1 contraction launches of a C2 PD solve (the
# constructor's canonicalisation is launch 0 of each sort-reduce kernel)
mkdir -p gpurun_out/ncu
for K in k_sr_count k_sr_scatter k_sr_tiles; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$K" -s 1 -c 1 \
    -o gpurun_out/ncu/r02_c2_contract_$K -f python tools/probe_configs.py c2 1 > gpurun_out/ncu/r02_c2_contract_$K.log 2>&1
  tail -1 gpurun_out/ncu/r02_c2_contract_$K.log
done
