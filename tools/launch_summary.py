"""Summarise an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv --log-file X` launch list: the kernels of the last
`--last` launches (one step), with time and DRAM bytes per kernel name.

usage: python tools/launch_summary.py launches.csv [--last K] [--json out.json]
"""
import argparse
import collections
import csv
import json
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--last", type=int, default=0)
    ap.add_argument("--after", default=None, help="only launches after the last launch of this kernel name")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    rows = [r for r in csv.DictReader(l for l in open(a.csv) if not l.startswith("=="))]
    launches = collections.OrderedDict()
    for r in rows:
        key = (r["ID"], re.sub(r"\(.*", "", r["Kernel Name"]).split("<")[0].split("::")[-1])
        launches.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    items = list(launches.items())
    if a.last:
        items = items[-a.last:]
    agg = collections.OrderedDict()
    for (_, name), m in items:
        t = agg.setdefault(name, {"us": 0.0, "dram_bytes": 0.0, "launches": 0})
        t["us"] += m.get("gpu__time_duration.sum", 0.0) / 1e3
        t["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        t["launches"] += 1
    tot = sum(v["us"] for v in agg.values())
    for k, v in agg.items():
        print(f"{k:28s} {v['us']:9.1f} us {v['us'] / tot * 100:5.1f}%  {v['dram_bytes'] / 1e6:9.1f} MB "
              f"{v['dram_bytes'] / max(v['us'], 1e-9) / 1e3:7.1f} GB/s  x{v['launches']}")
    print(f"{'total':28s} {tot:9.1f} us")
    if a.json:
        json.dump({"kernels": agg, "total_us": tot}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
