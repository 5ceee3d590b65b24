"""Summarise a tools/gemm_trace.py timeline: per mark, min / median / max over the CTAs that reached it."""
import statistics
import sys

for path in sys.argv[1:]:
    lines = open(path).read().splitlines()
    hdr = lines[1].split()
    rows = []
    for ln in lines[2:]:
        parts = ln.split()
        if not parts or not parts[0].isdigit():
            continue
        rows.append(parts)
    print(f"{path}: {lines[0]}  ({len(rows)} CTAs)")
    for j, name in enumerate(hdr[1:17], start=1):
        vals = [float(r[j]) for r in rows if j < len(r) and r[j] != "-"]
        if vals:
            print(f"  {name:>9}: min {min(vals):7.2f}  med {statistics.median(vals):7.2f}  max {max(vals):7.2f}  (n={len(vals)})")
