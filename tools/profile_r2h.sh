#!/bin/bash
# Round-2 final profiles on the GPU box: default bench line, its ncu launch list, and
# `ncu --set full` of the cfg4 and cfg3 SSPI chains on the fp16x3 CTA-pair engine.
#   gpurun -- 'bash tools/profile_r2h.sh r2h'
tag=${1:-r2h}
out=gpurun_out
mkdir -p $out
timeout 900 python bench.py > $out/${tag}_bench_cfg4_default.jsonl 2> $out/${tag}_bench_cfg4_default.err || exit 1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/${tag}_launches_cfg4_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-variants \
  > $out/${tag}_launches_ncu.log 2>&1
echo "launches rc=$?"
full() {   # name workload frames
  local cmd="python tools/prof_chain.py --workload $2 --variant sspi --frames $3 --reps 2 --engine tile_f16"
  timeout 600 $cmd || return 1
  timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:frontend|gather_pair|untile" -s 3 -c 3 \
    -o $out/${tag}_full_$1 -f $cmd > $out/${tag}_full_$1.log 2>&1
  ncu -i $out/${tag}_full_$1.ncu-rep --page raw --csv > $out/${tag}_full_$1_raw.csv
  echo "$1 rc=$?"
}
full cfg4_sspi cfg4 10000
full cfg3_sspi cfg3 10000
python tools/ncu_traffic.py --merge=profiles/traffic.json cfg4:sspi:$out/${tag}_full_cfg4_sspi_raw.csv \
  cfg3:sspi:$out/${tag}_full_cfg3_sspi_raw.csv > $out/traffic.json
rm -f $out/${tag}_full_cfg3_sspi.ncu-rep
ls -la $out | tail -12
