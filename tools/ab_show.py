import json, sys
for f in sys.argv[1:]:
    for l in open(f):
        if l.startswith('{'):
            d = json.loads(l)
            r = d['roofline']
            print(f.split('/')[-1], round(d['value'] / 1e6, 2), round(d['ms_per_step'], 3),
                  {k: round(v, 3) for k, v in d['stages_ms_per_step'].items()}, 'frac', round(r['frac'], 3),
                  'hits', r.get('memo_hits_per_step'), 'comp', r['compressions_per_step'],
                  'e2e', round(d['e2e']['value'] / 1e6, 2))
