"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, time, share."""
import csv, collections, sys
path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
r = csv.reader(lines)
hdr = next(r)
iN, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for row in r:
    name = row[iN].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(row[iV].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':58s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:58]:58s} {v[0]:8d} {v[1]/1e6:10.3f} {v[1]/v[0]/1e3:9.2f} {v[1]/tot:6.3f}")
print(f"total {tot/1e6:.3f} ms")
