"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum
--clock-control none --csv`) into per-kernel launch counts, total time and
share of the captured run.

    python profiles/launch_summary.py profiles/r01/launch_list_512.csv "<command>" > profiles/r01/launch_list_512_summary.txt
"""

import csv
import sys
from collections import defaultdict


def main(path, command):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        unit = r[ix["Metric Unit"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        ms = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}[unit]
        name = r[ix["Kernel Name"]].split("(")[0].strip()
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(t for _, t in agg.values())
    lines = ["# ncu launch list summary (gpu__time_duration.sum, --clock-control none, cold-cache serialised launches)",
             f"# command: {command}", "# kernel  launches  total_ms  share"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k:28s} {n:5d} {t:10.3f} {t / tot:7.3f}")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
