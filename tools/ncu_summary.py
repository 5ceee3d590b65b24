"""Per-launch summary of an ncu report (read here, no GPU needed):
    python tools/ncu_summary.py REPORT.ncu-rep [--algo-bytes N ...] > profiles/....json
Duration, DRAM read/write, achieved DRAM GB/s, tensor-pipe and SM throughput per launch."""

import argparse
import csv
import io
import json
import subprocess

METRICS = {"gpu__time_duration.sum": "duration_us", "dram__bytes_read.sum": "dram_read_B",
           "dram__bytes_write.sum": "dram_write_B", "launch__grid_size": "grid",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct", "lts__t_sector_hit_rate.pct": "l2_hit_pct",
           "launch__registers_per_thread": "regs"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        d = dict(zip(head, r))
        rec = {"kernel": d.get("Kernel Name", "")[:90]}
        for m, k in METRICS.items():
            if m not in d:
                continue
            try:
                rec[k] = float(d[m].replace(",", "")) * UNIT.get(units[head.index(m)], 1)
            except ValueError:
                rec[k] = d[m]
        if "duration_us" in rec and "dram_read_B" in rec:
            rec["dram_GBps"] = (rec["dram_read_B"] + rec.get("dram_write_B", 0)) / (rec["duration_us"] * 1e-6) / 1e9
        out.append(rec)
    print(json.dumps({"source": a.rep, "note": a.note, "launches": out}, indent=1))


if __name__ == "__main__":
    main()
