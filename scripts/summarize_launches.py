import csv, collections, sys
path = sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/ll_launches.csv'
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
h, d = rows[hi], rows[hi + 1:]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in d:
    name = r[ki].split('(')[0].replace('void ', '').split('<')[0].strip().replace('vmps::', '')
    v = float(r[vi].replace(',', ''))
    v *= {'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0}.get(r[ui], 1e-6)
    agg[name][0] += 1
    agg[name][1] += v
ours = {k: v for k, v in agg.items() if k.startswith('k_') or k.startswith('k4_')}
tot = sum(v[1] for v in ours.values())
print(f'{"kernel":34s} {"launches":>8s} {"ms":>10s} {"share":>7s}')
for k, (c, t) in sorted(ours.items(), key=lambda x: -x[1][1]):
    print(f'{k:34s} {c:8d} {t:10.3f} {t / tot * 100:6.1f}%')
print(f'{"total":34s} {sum(v[0] for v in ours.values()):8d} {tot:10.3f}')
