#!/bin/bash
# Round-end GPU tests + smoke + default bench (tools/final_check.sh), then an
# `ncu --set full` capture of the 4-frame untile pass at cfg4.
#   gpurun -- 'bash tools/profile_r1k.sh'
tag=r1k; out=gpurun_out; mkdir -p $out
bash tools/final_check.sh
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:untile" -s 1 -c 1 -o $out/${tag}_full_cfg4_untile -f \
  python tools/prof_chain.py --workload cfg4 --variant sspi --frames 10000 --reps 2 > $out/${tag}_full_cfg4_untile.log 2>&1
echo "ncu rc=$?"
ncu -i $out/${tag}_full_cfg4_untile.ncu-rep --page raw --csv > $out/${tag}_full_cfg4_untile_raw.csv
rm -f $out/${tag}_full_cfg4_untile.ncu-rep
python tools/ncu_summary.py $out/${tag}_full_cfg4_untile_raw.csv > $out/${tag}_ncu_summary.md
