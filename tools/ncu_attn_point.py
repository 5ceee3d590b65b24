"""Summarise an ncu --set full capture of k_decode_attn into profiles/attention_dram_bytes.json.

    python tools/ncu_attn_point.py gpurun_out/prof_attn_b384_c1400.ncu-rep --b 384 --ctx 1400 \
        --model qwen2.5-1.5b --workload C2

DRAM read + write bytes per launch (`traffic` of the bench line), the kernel duration and the
algorithmic bytes of the same launches (sum_rows ctx * KV bytes per token per layer
+ q / out), so the bench reports the traffic of the operating point it states.
"""

import argparse
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
           "launch__registers_per_thread"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--b", type=int, required=True)
    ap.add_argument("--ctx", type=int, required=True)
    ap.add_argument("--model", default="qwen2.5-1.5b")
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--out", default="profiles/attention_dram_bytes.json")
    a = ap.parse_args()
    import paper_2509_18521_b200 as pb

    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    launches = []
    for r in data:
        d = dict(zip(head, r))
        if "k_decode_attn" not in d.get("Kernel Name", ""):
            continue
        rec = {}
        for m in METRICS:
            if m in d:
                u = units[head.index(m)]
                try:
                    rec[m] = float(d[m].replace(",", "")) * UNIT.get(u, 1)
                except ValueError:
                    rec[m] = d[m]
        launches.append(rec)
    spec = pb.PRESETS[a.model]
    kv_tok_layer = 2 * spec.n_kv_heads * spec.head_dim * 2
    alg = a.b * a.ctx * kv_tok_layer + a.b * spec.n_q_heads * spec.head_dim * 2 * 2
    traffic = [x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in launches]
    dur = [x["gpu__time_duration.sum"] for x in launches]
    out = {"note": f"ncu --set full --clock-control none, k_decode_attn at the bench's average C2 operating point "
                   f"(b = {a.b} live rows, ctx = {a.ctx} per row; {a.model}, one layer per launch), "
                   f"tools/decode_microbench.py", "workload": a.workload, "point": {"b": a.b, "ctx": a.ctx},
           "bytes_per_launch": sum(traffic) / len(traffic), "algorithmic_bytes_per_launch": alg,
           "duration_us": dur, "dram_GBps": [t / (d * 1e-6) / 1e9 for t, d in zip(traffic, dur)],
           "launches": launches}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "launches"}, indent=1))


if __name__ == "__main__":
    main()
