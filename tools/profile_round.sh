#!/bin/bash
# On the GPU box: launch list of the default bench + `ncu --set full` of each hot kernel.
#   gpurun -- 'bash tools/profile_round.sh r1d'
# Every profiled command is first run once without ncu (it must exit 0).
tag=${1:-r1}
out=gpurun_out
mkdir -p $out
full() {   # name workload variant kernel-regex frames [skip count] [engine]
  local name=$1 wl=$2 var=$3 rx=$4 fr=$5 eng=${8:-auto}
  timeout 600 python tools/prof_chain.py --workload $wl --variant $var --frames $fr --reps 2 --engine $eng || return 1
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s ${6:-2} -c ${7:-2} \
    -o $out/${tag}_full_${name} -f python tools/prof_chain.py --workload $wl --variant $var --frames $fr --reps 2 \
    --engine $eng > $out/${tag}_full_${name}.log 2>&1
  ncu -i $out/${tag}_full_${name}.ncu-rep --page raw --csv > $out/${tag}_full_${name}_raw.csv
  echo "$name rc=$?"
}
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $out/${tag}_launch_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/${tag}_launches_cfg2_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  > $out/${tag}_launches_ncu.log 2>&1
echo "launches rc=$?"
full cfg2_sspi cfg2 sspi "frontend_map" 1000 1 2 fused
full cfg3_sspi cfg3 sspi "frontend|sspi|interp_tc" 10000
full cfg3_slri cfg3 slri "frontend|gemm|splitk|interp_tc|split_bf16" 10000 5 5
full cfg3_conv cfg3 conv "frontend|conv_gen" 10000
full cfg4_sspi cfg4 sspi "frontend|gather_tc|untile" 10000 3 3
python tools/ncu_traffic.py cfg2:sspi:$out/${tag}_full_cfg2_sspi_raw.csv cfg3:sspi:$out/${tag}_full_cfg3_sspi_raw.csv \
  cfg3:slri:$out/${tag}_full_cfg3_slri_raw.csv cfg3:conv:$out/${tag}_full_cfg3_conv_raw.csv \
  cfg3:conv_h:profiles/r1c_full_cfg3_conv_h_raw.csv cfg4:sspi:$out/${tag}_full_cfg4_sspi_raw.csv > $out/traffic.json
rm -f $out/${tag}_full_cfg4_sspi.ncu-rep $out/${tag}_full_cfg3_slri.ncu-rep $out/${tag}_full_cfg3_sspi.ncu-rep \
  $out/${tag}_full_cfg3_conv.ncu-rep
ls -la $out | tail -30
