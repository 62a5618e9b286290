#!/bin/bash
# On the GPU box: `ncu --set full` of the cfg3 SSPI chain (fp16x3 gathered windows, grid-order stores).
tag=${1:-r2f}
out=gpurun_out
mkdir -p $out
cmd="python tools/prof_chain.py --workload cfg3 --variant sspi --frames 10000 --reps 2 --engine ${2:-tile_f16}"
timeout 600 $cmd || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:frontend|gather_pair|untile" -s 2 -c 2 \
  -o $out/${tag}_full_cfg3_sspi -f $cmd > $out/${tag}_full_cfg3_sspi.log 2>&1
ncu -i $out/${tag}_full_cfg3_sspi.ncu-rep --page raw --csv > $out/${tag}_full_cfg3_sspi_raw.csv
ls -la $out | tail -5
