#!/bin/bash
# On the GPU box: `ncu --set full` of the cfg4 chain's kernels on the fp16x3 engine (fixed fit).
#   gpurun -- 'bash tools/profile_r2e.sh r2e'
tag=${1:-r2e}
out=gpurun_out
mkdir -p $out
cmd="python tools/prof_chain.py --workload cfg4 --variant sspi --frames 10000 --reps 2 --engine ${2:-tile_f16}"
timeout 600 $cmd || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:frontend|gather_pair|untile" -s 3 -c 3 \
  -o $out/${tag}_full_cfg4_sspi -f $cmd > $out/${tag}_full_cfg4_sspi.log 2>&1
ncu -i $out/${tag}_full_cfg4_sspi.ncu-rep --page raw --csv > $out/${tag}_full_cfg4_sspi_raw.csv
ls -la $out | tail
