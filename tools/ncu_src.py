"""Summarise an ncu report's source page: per SASS opcode (sass) or per CUDA
source line (cuda) the executed warp instructions and warp-stall samples.
Profiling helper only (reads a .ncu-rep here, no GPU).

usage: python tools/ncu_src.py REPORT KERNEL_REGEX [sass|cuda] [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
mode = sys.argv[3] if len(sys.argv) > 3 else "sass"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "sass" if mode == "sass" else "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0, 0])
tot = [0, 0]
fname = ""
cols = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if "Instructions Executed" in r:
        cols = (r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)"))
        continue
    if cols is None or len(r) <= cols[0]:
        continue
    if mode == "sass":
        src = r[cols[0] - 6].strip() if False else None
    try:
        ie, st = int(r[cols[0]] or 0), int(r[cols[1]] or 0)
    except ValueError:
        continue
    if mode == "sass":
        ins = r[1].strip().split()
        if not ins:
            continue
        op = ins[1] if ins[0].startswith("@") and len(ins) > 1 else ins[0]
        key = op.split(".")[0]
    else:
        if not r[0]:
            continue  # SASS rows under a CUDA line
        key = f"{fname}:{r[0]}: {r[1].strip()[:100]}"
    agg[key][0] += ie
    agg[key][1] += st
    tot[0] += ie
    tot[1] += st
print(f"total warp-instr {tot[0]:,}  stall samples {tot[1]:,}")
for k, (ie, st) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{ie:>13,} {100*ie/max(tot[0],1):5.1f}%  stall {100*st/max(tot[1],1):5.1f}%  {k}")
