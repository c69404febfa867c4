"""Top SASS lines by warp-stall samples of an ncu --set full report (run here).
    python tools/ncu_top_stalls.py report.ncu-rep [n]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iw = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[iw] or 0), r[ia], r[isrc]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print("total samples", tot)
for d in sorted(data, reverse=True)[:top]:
    print(f"{d[0]:6d} {100 * d[0] / tot:5.1f}%  {d[1]}  {d[2][:100]}")
