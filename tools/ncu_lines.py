#!/usr/bin/env python
"""Per-source-line warp-stall samples of an ncu `--page source --print-source cuda,sass --csv`
export (lines whose "Line No" is set carry the line's totals). Usage:
  ncu -i X.ncu-rep --page source --print-source cuda,sass --csv > x.csv; python tools/ncu_lines.py x.csv [top]"""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hdr]
    samp = h.index("# Samples")
    inst = h.index("Instructions Executed")
    out = []
    for r in rows[hdr + 1:]:
        if r and r[0].strip().isdigit():
            try:
                out.append((int(r[samp]), int(r[inst]), int(r[0]), r[1].strip()))
            except ValueError:
                pass
    tot = sum(o[0] for o in out) or 1
    print(f"total samples {tot}")
    for s, i, ln, src in sorted(out, reverse=True)[:top]:
        print(f"{s:8d} {100.0 * s / tot:5.1f}%  inst {i:10d}  L{ln:<5d} {src[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
