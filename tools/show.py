import json, sys
for f in sys.argv[1:]:
    try:
        for l in open(f):
            if l.startswith('{'):
                d = json.loads(l)
                print(f, round(d['value'] / 1e6, 1), 'Mrays/s', 'walk_ms', round(d['roofline']['avg_launch_ms'], 4),
                      'frac', round(d['roofline']['frac'], 3), 'ms/step', round(d['ms_per_step'], 3),
                      d.get('stages_ms_per_step'))
    except FileNotFoundError:
        print(f, 'missing')
