import sys, json, glob
for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/bench*.log')):
    for l in open(f):
        if l.startswith('{'):
            d = json.loads(l)
            print(f.split('/')[-1], round(d['value']), round(d['ms_per_step'], 1), round(d['achieved_hbm_gbs']), d['config'].get('kernels'), d['config'].get('prefetch'), {k: (round(v['ms'], 1), round(v['gbs'])) for k, v in d['kernels'].items()})
            break
    else:
        print(f, open(f).read()[-600:])
