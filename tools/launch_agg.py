"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel totals of the
second half of the launches (the last of two identical calls), and the k_fit3 launch times."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, recs = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            recs.append((d["Kernel Name"][:60], float(d["Metric Value"].replace(",", ""))))
half = recs[len(recs) // 2:]
agg = collections.defaultdict(lambda: [0, 0.0])
for k, v in half:
    agg[k][0] += 1
    agg[k][1] += v
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:4d} {t / 1e3:9.1f} us  {k}")
print("k_fit3 us:", [round(v / 1e3) for k, v in half if "k_fit3" in k])
