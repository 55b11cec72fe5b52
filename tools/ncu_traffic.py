"""Write profiles/ncu_traffic.json (per-kernel DRAM bytes per launch, read by
bench.py's roofline `traffic`) from an `ncu --set full` report of one step.

usage: python tools/ncu_traffic.py REPORT "SOURCE DESCRIPTION" [OUT]
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

rep, src = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_traffic.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
name_i = hdr.index("Kernel Name")
rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
acc = collections.defaultdict(list)
for r in rows[2:]:
    m = re.search(r"(k_[A-Za-z0-9_]+)", r[name_i])
    if not m:
        continue
    b = float(r[rd].replace(",", "")) * scale.get(units[rd], 1) + float(r[wr].replace(",", "")) * scale.get(units[wr], 1)
    acc[m.group(1)].append(b)
kern = {k: sum(v) / len(v) for k, v in acc.items()}
json.dump({"source": src, "kernels": kern}, open(out, "w"), indent=1)
print(json.dumps(kern, indent=1))
