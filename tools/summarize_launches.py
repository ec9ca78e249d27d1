"""Summarise an ncu launch-list CSV (gpu__time_duration.sum [+ dram bytes]) per kernel.

usage: python tools/summarize_launches.py <launches.csv> [title]
"""
import csv
import re
import sys
from collections import OrderedDict


def short(name: str) -> str:
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\(.*$", "", name) if not name.startswith("cub::") else name.split("(")[0]
    return name.replace("l0s::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    per = OrderedDict()
    seen = {}
    for r in rows:
        k = short(r["Kernel Name"])
        d = per.setdefault(k, {"ids": set(), "ns": 0.0, "dram": 0.0})
        d["ids"].add(r["ID"])
        val = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            scale = {"ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1.0}.get(unit, 1.0)
            d["ns"] += val * scale
        elif r["Metric Name"].startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d["dram"] += val * scale
        seen[k] = True
    search = sum(d["ns"] for k, d in per.items() if "dfma_peak" not in k and "rcp_check" not in k)
    print(f"# {title}")
    print("# kernel | launches | total ms | share of search time | DRAM bytes per launch (MB)")
    for k, d in sorted(per.items(), key=lambda kv: -kv[1]["ns"]):
        n = len(d["ids"])
        share = "" if ("dfma_peak" in k or "rcp_check" in k) else f"{100 * d['ns'] / search:5.1f}%"
        print(f"{k[:48]:48s} {n:5d} {d['ns'] / 1e6:9.3f} {share:>7s} {d['dram'] / n / 1e6:10.2f}")


if __name__ == "__main__":
    main()
