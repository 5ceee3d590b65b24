"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel (and grid)
launch count, total and average device time and share of the window.

    python tools/launch_summary.py gpurun_out/launches.csv
"""

import collections
import csv
import re
import sys


def summarise(path):
    rows = list(csv.DictReader(line for line in open(path) if line.startswith('"')))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").replace("unnamed>::", "")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3}.get(r["Metric Unit"], 1e-3)
        k = (name, r["Grid Size"])
        agg[k][0] += 1
        agg[k][1] += float(r["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = [f"# {path}: {sum(v[0] for v in agg.values())} launches, {tot / 1e3:.3f} ms total device time"]
    out.append(f"{'share':>6} {'launches':>8} {'avg_us':>9}  kernel  grid")
    for (name, grid), (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{100 * us / tot:5.1f}% {n:8d} {us / n:9.1f}  {name}  {grid}")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarise(p))
