"""Last-run view of an ncu launch list: per-kernel totals over the kernels after
the (runs-1)-th k_reset.  usage: launch_tail.py list.csv [runs]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; ik = h.index('Kernel Name'); iv = h.index('Metric Value')
ks = []
for r in rows[hdr + 1:]:
    if len(r) > iv:
        ks.append((r[ik].split('(')[0].replace('void ', ''), float(r[iv].replace(',', '')) / 1e3))
resets = [i for i, (n, _) in enumerate(ks) if n.startswith('k_reset')]
tail = ks[resets[runs - 1]:] if len(resets) >= runs else ks
tot, cnt = {}, {}
for n, v in tail:
    tot[n] = tot.get(n, 0) + v
    cnt[n] = cnt.get(n, 0) + 1
s = sum(tot.values())
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{n[:48]:48s} {v:10.1f} us {100 * v / s:5.1f}% {cnt[n]:5d}  {v / cnt[n]:8.2f} us/launch")
print(f"{'total':48s} {s:10.1f} us")
