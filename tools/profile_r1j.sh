#!/bin/bash
# Final-state `ncu --set full` captures of the kernels changed late in the round:
# cfg4 tile engine (task-per-warp frontend, round-robin gather, untile), cfg2 split-K
# conventional map, cfg3 SLRI / LR (8-epilogue-warp candidate product, narrow GEMM).
#   gpurun -- 'bash tools/profile_r1j.sh'
tag=r1j; out=gpurun_out; mkdir -p $out
cap() {  # name workload variant regex frames skip count
  timeout 600 python tools/prof_chain.py --workload $2 --variant $3 --frames $5 --reps 2 || return 1
  timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$4" -s $6 -c $7 -o $out/${tag}_full_$1 -f \
    python tools/prof_chain.py --workload $2 --variant $3 --frames $5 --reps 2 > $out/${tag}_full_$1.log 2>&1
  ncu -i $out/${tag}_full_$1.ncu-rep --page raw --csv > $out/${tag}_full_$1_raw.csv
  rm -f $out/${tag}_full_$1.ncu-rep
  echo "$1 rc=$?"
}
cap cfg2_conv cfg2 conv "conv_gen|splitk" 1000 2 2
cap cfg3_slri cfg3 slri "interp_tc|gemm_nt" 10000 2 2
cap cfg3_lr cfg3 lr "interp_tc|gemm_nt" 10000 3 3
cap cfg4_sspi cfg4 sspi "frontend_lane|gather_tc|untile" 10000 3 3
python tools/ncu_traffic.py cfg2:sspi:profiles/r1g_full_cfg2_sspi_fused_raw.csv \
  cfg2:conv:$out/${tag}_full_cfg2_conv_raw.csv cfg3:sspi:profiles/r1e_full_cfg3_sspi_raw.csv \
  cfg3:slri:$out/${tag}_full_cfg3_slri_raw.csv cfg3:lr:$out/${tag}_full_cfg3_lr_raw.csv \
  cfg3:conv:profiles/r1e_full_cfg3_conv_raw.csv cfg3:conv_h:profiles/r1c_full_cfg3_conv_h_raw.csv \
  cfg4:sspi:$out/${tag}_full_cfg4_sspi_raw.csv > $out/traffic.json
ls -la $out | grep $tag
