import signal
signal.signal(signal.SIGPIPE, signal.SIG_DFL)
import json,sys
for f in sys.argv[1:]:
    d=json.loads(open(f).read().strip().split('\n')[-1])
    print(f, 'value', round(d['value'],2), 'ms/step', round(d['ms_per_step'],3), 'N', d['n_unique'], 'it', d['iterations'], 'flag', d['flagged_per_step'], 'swept', round(d.get('swept_fraction') or 0, 3), 'lloyd d/s %.3g'%d['lloyd_distances_per_s'], 'launches', d['gpu_launches'])
    print('  stages', {k: round(v,3) for k,v in d['stage_ms_last_step'].items()})
    print('  kernels', {k: (round(v['ms_per_step'],3), v['launches_per_step']) for k,v in d['kernels'].items()})
    r=d['roofline']; print('  roofline %s frac %.3f achieved %.2f avg_launch_ms %.4f share %.3f'%(r['kernel'][:24], r['frac'] or 0, r['achieved'] or 0, r['avg_launch_ms'], r['launch_share_of_step']), 'e2e', d['e2e']['value'] if d['e2e'] else None)
    if 'sweep_isolated' in r: print('  sweep_isolated', {k: round(v,4) for k,v in r['sweep_isolated'].items()})
    print('  bytek', {k:round(v['achieved_gbs'] or 0,1) for k,v in d['byte_kernels'].items()}, 'clocks', d['clocks'])
