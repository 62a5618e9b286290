#!/bin/bash
# Final-state captures: launch list of the default bench, ncu --set full of the fused
# SSPI / SLRI chains at cfg2 and of the split-K conventional map at cfg2.
#   gpurun -- 'bash tools/profile_r1g.sh'
tag=r1g; out=gpurun_out; mkdir -p $out
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-variants > $out/${tag}_launch_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/${tag}_launches_cfg2_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-variants \
  > $out/${tag}_launches_ncu.log 2>&1
echo "launches rc=$?"
cap() {  # name variant regex engine
  timeout 300 python tools/prof_chain.py --workload cfg2 --variant $2 --frames 1000 --reps 2 --engine $4 || return 1
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$3" -s 1 -c 1 -o $out/${tag}_full_$1 -f \
    python tools/prof_chain.py --workload cfg2 --variant $2 --frames 1000 --reps 2 --engine $4 > $out/${tag}_full_$1.log 2>&1
  ncu -i $out/${tag}_full_$1.ncu-rep --page raw --csv > $out/${tag}_full_$1_raw.csv
  ncu -i $out/${tag}_full_$1.ncu-rep --page source --csv --print-source cuda,sass > $out/${tag}_full_$1_src.csv 2>/dev/null
  echo "$1 rc=$?"
}
cap cfg2_sspi_fused sspi "frontend_map" fused
cap cfg2_slri_fused slri "frontend_map" fused
cap cfg2_conv_splitk conv "conv_gen|splitk" auto
ls -la $out | grep $tag
