"""Per-source-line summary of an ncu report captured with --import-source on:
  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X_cs.csv
  python tools/ncu_lines.py X_cs.csv [top]
Prints the lines with the most stall samples and executed warp instructions, with the average
active threads per instruction of each line (the kernel's divergence by source line)."""
import csv
import os
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    cur = None
    hdr = None
    lines = []
    for r in csv.reader(open(path, newline="")):
        if len(r) == 2 and r[0] == "File Path":
            cur = os.path.basename(r[1])
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and len(r) == len(hdr) and r[0] != "":
            d = dict(zip(hdr[4:], r[4:]))
            lines.append((cur, int(r[0]), r[1].strip(), int(d["# Samples"] or 0), int(d["Instructions Executed"] or 0),
                          int(d["Thread Instructions Executed"] or 0)))
    ts = sum(x[3] for x in lines) or 1
    ti = sum(x[4] for x in lines) or 1
    tt = sum(x[5] for x in lines)
    print(f"total samples {ts}, warp instructions {ti}, avg threads/inst {tt / ti:.2f}")
    byfile = {}
    for f, _, _, s, i, t in lines:
        a = byfile.setdefault(f, [0, 0, 0])
        a[0] += s
        a[1] += i
        a[2] += t
    print("\nper file: samples%  inst%  threads/inst")
    for f, a in sorted(byfile.items(), key=lambda kv: -kv[1][0]):
        print(f"  {f:28s} {100 * a[0] / ts:5.1f} {100 * a[1] / ti:5.1f} {a[2] / max(a[1], 1):5.1f}")
    print(f"\ntop {top} lines by stall samples: samples% inst% threads/inst  file:line  source")
    for f, ln, src, s, i, t in sorted(lines, key=lambda x: -x[3])[:top]:
        print(f"  {100 * s / ts:5.1f} {100 * i / ti:5.1f} {t / max(i, 1):5.1f}  {f}:{ln}  {src[:90]}")


if __name__ == "__main__":
    main()
