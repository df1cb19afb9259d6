import glob, json, sys
for f in sorted(glob.glob(sys.argv[1])):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d['roofline']
        print(f"{f:40s} {d['value']:.3e} ms/step {d['ms_per_step']:.4f} frac {r['frac']:.3f} ach {r['achieved']:.0f} share {r['pass_share_of_step']:.2f} clk {d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')}")
    except Exception as e:
        print(f, 'ERR', e, open(f.replace('.json', '.err')).read()[-300:])
