#!/usr/bin/env python
"""Summary of a dataflow-sweep trace (trace build, PSCU_FLOW_TRACE=<prefix>):
per task globaltimer stamps {start, operands loaded, sources arrived,
folded}. Prints the sweep span, the per-level advance of the latest finish,
and where a task's time goes (operand loads, waiting for sources, fold).
Usage: python tools/analyze_flow_trace.py gpurun_out/ft_fwd.bin"""
import sys

import numpy as np


def load(path):
    raw = open(path, "rb").read()
    nsub, ntt = np.frombuffer(raw[:16], np.int64)
    hdr = np.frombuffer(raw[16:16 + 4 * 16 * nsub], np.int32).reshape(nsub, 16)
    body = raw[16 + 4 * 16 * nsub:]
    stride = len(body) // (8 * ntt)  # 4 (stamps) or 6 (+ fold cycles, lane-parallel flag)
    st = np.frombuffer(body[:8 * ntt * stride], np.int64).reshape(ntt, stride)
    return hdr, st


def main(path):
    hdr, st = load(path)
    rows = []
    for ch in range(len(hdr)):
        nt, t0 = int(hdr[ch, 8]), int(hdr[ch, 9])
        s = st[t0:t0 + nt]
        s = s[s[:, 3] > 0]
        if len(s):
            rows.append((ch, len(s), s[:, 0].min(), s[:, 3].max(), np.mean(s[:, 1] - s[:, 0]),
                         np.mean(s[:, 2] - s[:, 1]), np.mean(s[:, 3] - s[:, 2]),
                         np.max(s[:, 3] - s[:, 2])))
    r = np.array(rows, dtype=float)
    t_begin, t_end = r[:, 2].min(), r[:, 3].max()
    adv = np.diff(r[:, 3])
    print(f"{path}: {len(r)} task levels, span {(t_end - t_begin) / 1e3:.1f} us, "
          f"{(t_end - t_begin) / len(r):.0f} ns per level")
    print(f"  latest-finish advance per level: median {np.median(adv):.0f} ns, "
          f"p90 {np.percentile(adv, 90):.0f} ns")
    print(f"  per task (mean over levels): operand loads {r[:, 4].mean():.0f} ns, "
          f"wait for sources {r[:, 5].mean():.0f} ns, fold {r[:, 6].mean():.0f} ns "
          f"(slowest fold per level {r[:, 7].mean():.0f} ns)")
    print(f"  tasks per level: median {np.median(r[:, 1]):.0f}")
    # the critical path level by level: the task that finishes a level last,
    # measured from the previous level's last finish
    lastf = []
    for ch in range(len(hdr)):
        nt, t0 = int(hdr[ch, 8]), int(hdr[ch, 9])
        s = st[t0:t0 + nt]
        s = s[s[:, 3] > 0]
        if len(s):
            lastf.append(s[np.argmax(s[:, 3])])
    lastf = np.array(lastf)
    if len(lastf) > 2:
        prev = lastf[:-1, 3]
        cur = lastf[1:]
        print(f"  level-closing task vs previous level's close: start {np.median(cur[:, 0] - prev):.0f} ns, "
              f"loads done {np.median(cur[:, 1] - prev):.0f} ns, sources in {np.median(cur[:, 2] - prev):.0f} ns, "
              f"folded {np.median(cur[:, 3] - prev):.0f} ns (medians)")
        if st.shape[1] >= 6:
            print(f"  level-closing task fold: {np.median(cur[:, 4]):.0f} cycles median")
    if st.shape[1] >= 6:
        done = st[st[:, 3] > 0]
        kinds = done[:, 5] % 1000
        if (done[:, 5] >= 1000).any():
            sel = done[:, 5] >= 1000
            a0 = (done[sel, 5] // 1000) % 100
            a1 = done[sel, 5] // 100000
            print(f"  shuffle-chain tasks: active lanes at entry median {np.median(a0):.0f} "
                  f"(min {a0.min()}), in the row loop median {np.median(a1):.0f} (min {a1.min()})")
        for name, sel in (("lane-parallel", kinds == 1), ("lane-0 leading in-task + chain", kinds == 2),
                          ("lane-0 general order", kinds == 0),
                          ("warp-replicated shuffle chain", kinds == 3),
                          ("lane-0 dense-product blocks", kinds == 4),
                          ("lane-per-row dense-product blocks", kinds == 5)):
            if sel.any():
                cyc = done[sel, 4]
                print(f"  {name} folds: {int(sel.sum())} tasks, {np.median(cyc):.0f} cycles median, "
                      f"p90 {np.percentile(cyc, 90):.0f}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
