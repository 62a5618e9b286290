for wl in cfg3 cfg2; do
  timeout 600 python bench.py --workload $wl --variant slri --steps 10 --warmup 3 --no-cpu-baseline --variants lr > gpurun_out/lrab_${wl}.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/lrab_${wl}.log').read().strip().splitlines()[-1]);print('$wl slri', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['parity']['max_normalized_error']); print({k:(v.get('ms_per_step'), v.get('parity',{}).get('max_normalized_error')) for k,v in d['variants'].items()})" || tail -3 gpurun_out/lrab_${wl}.log
done
