for wl in cfg4; do for d in 2; do
  fr=""; [ $wl = cfg4 ] && fr="--frames 2000"
  SRPGPU_SSPI_DIRECT=$d timeout 400 python bench.py --workload $wl $fr --steps 5 --warmup 3 --no-cpu-baseline --variants sspi > gpurun_out/ab_${wl}_$d.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_${wl}_$d.log').read().strip().splitlines()[-1]);print('$wl direct=$d', d['ms_per_step'], d['roofline']['kernel_ms'], d.get('parity',{}).get('max_normalized_error') if isinstance(d.get('parity'),dict) else d.get('parity'))" || tail -3 gpurun_out/ab_${wl}_$d.log
done; done
