# ncu --set full captures of the kernels added late in round 2 (C2, first launch of each)
O=gpurun_out/ncu_late; mkdir -p $O
cap() {  # label regex skip
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 1 \
    -o $O/r02_c2_$1 -f python tools/probe_configs.py c2 1 > $O/$1.log 2>&1
  tail -1 $O/$1.log
}
cap k_tri_out_handles "^k_tri_out_handles" 0
cap k_tri_kinds "^k_tri_kinds" 0
cap k_tree_resolve "^k_tree_resolve" 0
cap k_crx_emit "^k_crx_emit" 0
cap k_fetch "k_fetch" 5
