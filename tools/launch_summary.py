"""Summarise an ncu --metrics gpu__time_duration.sum launch list: time per kernel family."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; ik = h.index('Kernel Name'); iv = h.index('Metric Value')
tot, cnt = {}, {}
for r in rows[hdr + 1:]:
    if len(r) <= iv:
        continue
    name = r[ik].split('(')[0].split('<')[0].replace('void ', '')
    v = float(r[iv].replace(',', '')) / 1e6
    tot[name] = tot.get(name, 0) + v
    cnt[name] = cnt.get(name, 0) + 1
s = sum(tot.values())
print(f"{'kernel':34s} {'ms':>9s} {'share':>6s} {'launches':>8s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:34s} {v:9.3f} {v / s * 100:5.1f}% {cnt[k]:8d}")
print(f"{'total':34s} {s:9.3f}")
