"""Per-block stall breakdown of an ncu source (SASS) page, grouped by execution count.

usage: python tools/ncu_blocks.py src.csv [N] [--dump EXEC]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ie = ix["Instructions Executed"]
b = collections.defaultdict(lambda: {"n": 0, "ni": 0, "st": collections.Counter(), "ops": collections.Counter()})
for r in data:
    n = int(r[ie] or 0)
    v = b[n]
    v["n"] += n
    v["ni"] += 1
    op = r[ix["Source"]].strip().split()
    op = [o for o in op if not o.startswith("@")]
    v["ops"][op[0].split(".")[0] if op else "?"] += 1
    for k in reasons:
        v["st"][k[6:]] += float(r[ix[k]] or 0)
tot_s = sum(sum(v["st"].values()) for v in b.values())
tot_i = sum(v["n"] for v in b.values())
if "--dump" in sys.argv:
    want = int(sys.argv[sys.argv.index("--dump") + 1])
    for r in data:
        if int(r[ie] or 0) == want:
            st = {k[6:]: float(r[ix[k]] or 0) for k in reasons if float(r[ix[k]] or 0) > 0}
            print(r[ix["Source"]][:70].ljust(70), sorted(st.items(), key=lambda x: -x[1])[:3])
    sys.exit()
for n, v in sorted(b.items(), key=lambda kv: -sum(kv[1]["st"].values()))[: int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 8]:
    s = sum(v["st"].values())
    top = ", ".join(f"{k} {c / s:.0%}" for k, c in v["st"].most_common(5))
    ops = ", ".join(f"{k}:{c}" for k, c in v["ops"].most_common(8))
    print(f"exec {n:>8} ninstr {v['ni']:>5} instr {v['n'] / tot_i:6.1%} stalls {s / tot_s:6.1%} | {top}\n      ops {ops}")
