"""Print raw ncu metrics whose names contain any of the given substrings.

usage: ncu -i X.ncu-rep --page raw --csv | python tools/ncu_raw_grep.py tensor lts__t_bytes ...
"""
import csv
import sys

rows = list(csv.reader(sys.stdin))
hdr, units, vals = rows[0], rows[1], rows[2]
for k, u, v in zip(hdr, units, vals):
    if any(s in k for s in sys.argv[1:]):
        print(f"{k:80s} {v} {u}")
