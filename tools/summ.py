import json, sys
for f in sys.argv[1:]:
    l=[x for x in open(f) if x.startswith('{')]
    if not l: print(f, open(f).read()[-1500:]); continue
    d=json.loads(l[-1])
    if d.get('impl') == 'reference':
        print(f, 'REF', d['value'], d.get('cpu_baseline', {}).get('sample')); continue
    r=d['roofline']
    print(f, d['config']['workload'], d['config'].get('map_engine'), 'value %.4g ms %.4f e2e %.4g launches %s' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches_per_step']))
    print('   roof %s frac %.3f kernel_ms %s eng %s' % (r['kernel'], r['frac'], {k: round(v, 4) for k, v in r['kernel_ms'].items()}, r.get('map_engine')))
    print('   parity', d['parity'].get('max_normalized_error'), d['parity'].get('argmax_agree_on_margin_frames'), 'clocks', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
    for k, v in d['variants'].items():
        print('   var %-6s %s' % (k, {kk: (round(vv, 5) if isinstance(vv, float) else vv) for kk, vv in v.items() if kk in ('value', 'ms_per_step', 'error', 'tflops_gemm')}), v.get('parity', {}).get('max_normalized_error'))
    if d.get('cpu_baseline'): print('   cpu', d['cpu_baseline'])
