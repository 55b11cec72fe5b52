"""Per-source-line summary of an ncu `--page source --csv --print-source cuda,sass` export.

usage: python tools/ncu_lines.py export.csv [top]
Prints the source lines with the most executed warp instructions and stall samples.
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    f = None
    out = []
    tot_i = tot_s = 0
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if len(r) > 7 and r[2] == "-" and r[0].isdigit():
            try:
                ins = int(r[7])
                smp = int(r[4])
            except ValueError:
                continue
            tot_i += ins
            tot_s += smp
            out.append((ins, smp, f, int(r[0]), r[1][:110]))
    print(f"total warp instructions {tot_i:,}  stall samples {tot_s:,}")
    for ins, smp, f, ln, src in sorted(out, reverse=True)[:top]:
        print(f"{ins / tot_i * 100:5.1f}% ins {smp / max(tot_s, 1) * 100:5.1f}% smp  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
