"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel name: total ms, launches, share.  Optional --after N skips the first N
launches (warm-up / calibration).

    python tools/launch_summary.py gpurun_out/launches.csv [--top 40] > profiles/<r>_launches_summary.md
"""

from __future__ import annotations

import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--after", type=int, default=0)
    a = ap.parse_args()
    rows = []
    with open(a.csv) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ms = v / 1e6 if unit in ("nsecond", "ns") else v / 1e3 if unit in ("usecond", "us") else v
        rows.append((int(r["ID"]), r["Kernel Name"], ms))
    rows = [x for x in rows if x[0] >= a.after]
    agg = collections.defaultdict(lambda: [0.0, 0])
    for _, name, ms in rows:
        agg[name][0] += ms
        agg[name][1] += 1
    tot = sum(v[0] for v in agg.values())
    print(f"total {tot:.1f} ms over {len(rows)} launches\n")
    print("| share | ms | launches | kernel |\n|---|---|---|---|")
    for name, (ms, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:a.top]:
        print(f"| {100 * ms / tot:.2f}% | {ms:.2f} | {n} | `{name[:100]}` |")


if __name__ == "__main__":
    main()
