import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print('value %.0f it/s  ms/step %.3f  launches %s' % (d['value'], d['ms_per_step'], d.get('gpu_launches')))
r = d['roofline']; print('roofline', {k: r[k] for k in ('kernel','variant','achieved','frac','traffic','ms_per_launch')})
for v, p in d['per_variant'].items():
    print('%-8s %6.1f us/it  %5.0f GB/s  frac %.3f' % (v, p['us_per_iter'], p['gbs'], p['roofline_frac']))
for k in d['kernels']:
    print('   %-8s %-7s %6.1f us %5.0f GB/s' % (k['variant'], k['kernel'], k['ms_per_launch']*1e3, k['gbs']))
print('e2e', d['e2e'] and round(d['e2e']['value']), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value'],1), 'clocks', d['clocks'])
