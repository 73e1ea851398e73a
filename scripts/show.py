import json, sys
for f in sys.argv[1:]:
    try:
        l = [x for x in open(f) if x.startswith('{')][0]
    except (IndexError, FileNotFoundError):
        print(f, "no result"); continue
    d = json.loads(l)
    print(f.split('/')[-1], d['config']['workload'], '%.4g' % d['value'], 'ms %.3f' % d['ms_per_step'],
          {k: round(v, 3) for k, v in d['breakdown_ms'].items()}, 'frac %.4f' % d['roofline']['frac'],
          'est %.3g/s' % d['estimate_evals_per_s'])
