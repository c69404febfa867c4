"""Per-step view of an ncu launch list (gpu__time_duration.sum): kernels between
two k_update* launches form one Greedy step.  usage: launch_steps.py list.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; ik = h.index('Kernel Name'); iv = h.index('Metric Value')
steps, cur = [], {}
for r in rows[hdr + 1:]:
    if len(r) <= iv:
        continue
    name = r[ik].split('(')[0].split('<')[0].replace('void ', '')
    v = float(r[iv].replace(',', '')) / 1e3  # us
    cur[name] = cur.get(name, 0.0) + v
    if name.startswith('k_update'):
        steps.append(cur); cur = {}
if cur:
    steps.append(cur)
names = sorted({k for s in steps for k in s}, key=lambda k: -sum(s.get(k, 0) for s in steps))[:8]
print('step ' + ' '.join(f'{n[:12]:>12s}' for n in names) + '    total(us)')
for i, s in enumerate(steps):
    print(f'{i:4d} ' + ' '.join(f'{s.get(n, 0):12.1f}' for n in names) + f' {sum(s.values()):12.1f}')
