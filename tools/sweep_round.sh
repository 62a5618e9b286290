#!/bin/bash
# On the GPU box: every workload's bench line (+ the reference arm) for DESIGN.md / profiles.
#   gpurun -- 'bash tools/sweep_round.sh r1'
tag=${1:-r1}; out=gpurun_out; mkdir -p $out
run() { local name=$1; shift; timeout 900 python bench.py "$@" > $out/${tag}_bench_${name}.log 2>&1; echo "$name rc=$?"; }
run cfg2 --steps 20 --warmup 5
run cfg2_ref --impl reference --steps 3 --warmup 3
run cfg1 --workload cfg1 --steps 20 --warmup 5 --no-cpu-baseline
run cfg3 --workload cfg3 --steps 10 --warmup 3 --variants sspi,slri,lr,conv,conv_h
run cfg4 --workload cfg4 --steps 3 --warmup 3 --variants conv
run cfg5 --workload cfg5 --steps 20 --warmup 5 --no-cpu-baseline
