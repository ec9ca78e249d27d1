"""Group an ncu source (SASS) page by execution count: where instructions and stall samples go.

usage: ncu -i X.ncu-rep --page source --csv --print-source sass > x.csv; python tools/sass_hot.py x.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ia = hdr.index("Instructions Executed")
iss = hdr.index("Warp Stall Sampling (All Samples)")
isrc = hdr.index("Source")
b = collections.defaultdict(lambda: [0, 0, 0, None])
for k, r in enumerate(data):
    n = int(r[ia] or 0)
    s = float(r[iss] or 0)
    v = b[n]
    v[0] += n
    v[1] += s
    v[2] += 1
    if v[3] is None:
        v[3] = k
tot = sum(v[0] for v in b.values())
ts = sum(v[1] for v in b.values())
for n, v in sorted(b.items(), key=lambda kv: -kv[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"exec {n:>9}  ninstr {v[2]:>5}  first@{v[3]:>5}  instr {v[0] / tot:6.1%}  stall-samples {v[1] / ts:6.1%}")
