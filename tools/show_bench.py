import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print('ttft', {k: round(v, 2) for k, v in d['ttft_ms'].items()}, 'roof', round(d['ttft_roofline']['roof_ms'], 2),
      'frac', round(d['ttft_roofline']['frac'], 3), 'rho', round(d['config']['rho'], 3))
print('sweep', {k: round(v, 2) for k, v in d['sweep_ms'].items()}, 'e2e', round(d['e2e']['value'], 2),
      'launches', d['gpu_launches'])
for k, v in d['kernels'].items():
    print(f"  {k:20s} {v['ms_per_step']:8.3f} ms x{v['launches_per_step']:5.0f}  TF/s {v['tflops'] and round(v['tflops'])}  GB/s {v['gbs'] and round(v['gbs'])}")
r = d['roofline']
print('roofline', r['kernel'], r['bound'], round(r['achieved']), r['peak'], round(r['frac'], 3))
print('clocks', d['clocks'], 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value']))
if d.get('decode'):
    x = d['decode']
    print('decode', {k: (round(v, 3) if isinstance(v, float) else v) for k, v in x.items() if k != 'note'})
if d.get('compute_bound_rho1'):
    print('rho1', {k: round(v, 3) for k, v in d['compute_bound_rho1'].items()})
