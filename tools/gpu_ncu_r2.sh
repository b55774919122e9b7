# Round-2 ncu --set full captures on C2 (one launch each; round-1 launch of
# the solve: the constructor's canonicalisation is launch 0 of the k_sr_* kernels)
mkdir -p gpurun_out/ncu2
cap() {  # label regex skip
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 1 \
    -o gpurun_out/ncu2/r02_c2_$1 -f python tools/probe_configs.py c2 1 > gpurun_out/ncu2/$1.log 2>&1
  tail -1 gpurun_out/ncu2/$1.log
}
cap k_sep_src "^k_sep_src" 0
cap k_cl_rounds "^k_cl_rounds" 0
cap k_mp_edge "^k_mp_edge" 0
cap k_mp_triplet "^k_mp_triplet" 0
cap k_sr_count "^k_sr_count" 1
cap k_sr_scatter "^k_sr_scatter" 1
cap k_sr_tiles "^k_sr_tiles" 1
cap k_match_vote "^k_match_vote" 0
cap k_bucket_scatter "^k_bucket_scatter" 0
cap k_rank_rows "^k_rank_rows" 0
cap k_reparam "^k_reparam" 0
