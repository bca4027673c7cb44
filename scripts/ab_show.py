import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "no result", e)
        continue
    r = d['roofline']
    o = d.get('online') or {}
    print(f.split('/')[-1], "step %.1f us" % (d['ms_per_step'] * 1e3),
          "dist %.1f us frac %.3f kern %.1f" % (r['kernel_ms'] * 1e3, r['frac'], (r.get('kernel_only_ms') or 0) * 1e3),
          "online %.1f busiest %.1f" % (o.get('round_us', 0), o.get('busiest_round_us', 0)),
          [(s['seed'], round(s['ms_per_step'] * 1e3, 1), round(s['distance_frac'], 3))
           for s in d.get('seed_stats', {}).get('per_seed', [])], (d.get('parity') or {}).get('ok'))
