"""Summaries of ncu output for profiles/.

  launches <csv> [out.md]   per-kernel totals of a `--metrics gpu__time_duration.sum` launch list
  full <csv> [kernel-substr] per-launch metrics of a `--set full --page raw --csv` export
"""
import csv
import io
import json
import re
import sys
from collections import defaultdict


def _rows(path):
    with open(path) as f:
        text = f.read()
    start = text.find('"ID"')
    return list(csv.DictReader(io.StringIO(text[start:])))


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    name = name.replace("<unnamed>::", "").replace("unnamed>::", "")
    return name


def launches(path, out=None):
    rows = _rows(path)
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        agg[k][0] += 1
        v = float(r["Metric Value"].replace(",", ""))
        agg[k][1] += v * (1e-3 if r["Metric Unit"] == "ns" else 1.0 if r["Metric Unit"] == "us" else 1e3)
    total = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {c} | {us:.1f} | {us / c:.2f} | {us / total:.1%} |")
    lines.append(f"| total | {sum(v[0] for v in agg.values())} | {total:.1f} | | 100% |")
    s = "\n".join(lines)
    if out:
        open(out, "w").write(s + "\n")
    print(s)
    return agg


def full(path, sub=""):
    rows = _rows(path)
    res = []
    for r in rows:
        if sub and sub not in r.get("Kernel Name", ""):
            continue
        res.append(r)
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]
    out = []
    for r in res:
        d = {"kernel": short(r.get("Kernel Name", "")), "grid": r.get("Grid Size"),
             "block": r.get("Block Size")}
        for k in keys:
            if k in r:
                d[k] = r[k]
        out.append(d)
    print(json.dumps(out, indent=1))
    return out


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
