set -x
mkdir -p gpurun_out
python bench.py --no-cpu-baseline --variants sspi,slri > gpurun_out/wpf_default.jsonl 2> gpurun_out/wpf_default.err
for r in 1 2; do
for w in 1 2 4; do
  for wl in cfg2 cfg1; do
    for v in sspi slri; do
      SRPGPU_FUSED_WPF=$w timeout 300 python bench.py --workload $wl --variant $v --no-cpu-baseline --no-variants --steps 40 2>>gpurun_out/wpf.err | sed "s/^/{\"wpf\": $w, \"r\": $r, \"line\": /; s/\$/}/" >> gpurun_out/wpf_ab.jsonl
    done
  done
done
done
