for wl in cfg2 cfg3; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/fab_${wl}.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/fab_${wl}.log').read().strip().splitlines()[-1]);print('$wl', d['ms_per_step'], d['roofline']['kernel_ms'], d['parity']['max_normalized_error'])" || tail -3 gpurun_out/fab_${wl}.log
done
