"""Run outputs in the reference's on-disk schema.

The reference CLI writes one directory per run (`cli.py:50-74`): `steps.jsonl` (one
`StepReport.to_json_dict()` per step, `metrics.py:24-51`), `summary.json` (`RunSummary` plus
`resolved_config`, keys sorted, `metrics.py:126-143`), optionally `samples.csv` (the delivered-sample
manifest, `simulate.py:90-103`) and `events.jsonl` (engine event records); `compare` adds
`comparison.json` over paired baseline / APRIL runs (`cli.py:83-129`).  Writing GPU runs in the same
schema lets the reference's metrics code and report frontend consume them unchanged
(`frontend/src/data.ts:6-22`).
"""

from __future__ import annotations

import json
import os

import numpy as np

from .metrics import RunSummary, StepReport

MANIFEST_HEADER = "step,instance_id,sample_index,start_version,complete_version,tokens\n"


def manifest_rows(step: int, batch) -> list[tuple]:
    """(step, instance_id, sample_index, start_version, complete_version, tokens) per delivered sample,
    in delivery order (simulate.py:90-103)."""
    rows = []
    for g in batch:
        for s in g.samples:
            rows.append((step, s.instance_id, s.sample_index, s.start_version, s.complete_version, s.total_tokens))
    return rows


def write_run_outputs(out_dir: str, reports: list[StepReport], summary: RunSummary | None, resolved_config: dict,
                      manifest: list[tuple] | None = None, events: list[dict] | None = None) -> None:
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "steps.jsonl"), "w", encoding="utf-8") as f:
        for r in reports:
            f.write(json.dumps(r.to_json_dict()) + "\n")
    s = summary.to_json_dict() if summary is not None else {"steps": 0}
    s["resolved_config"] = resolved_config
    with open(os.path.join(out_dir, "summary.json"), "w", encoding="utf-8") as f:
        json.dump(s, f, indent=2, sort_keys=True)
        f.write("\n")
    if manifest is not None:
        with open(os.path.join(out_dir, "samples.csv"), "w", encoding="utf-8") as f:
            f.write(MANIFEST_HEADER)
            for row in manifest:
                f.write(",".join(str(x) for x in row) + "\n")
    if events is not None:
        with open(os.path.join(out_dir, "events.jsonl"), "w", encoding="utf-8") as f:
            for rec in events:
                f.write(json.dumps(rec) + "\n")


def comparison_record(per_seed: list[dict], resolved_config: dict) -> dict:
    """`per_seed` entries: {"seed", "baseline": summary dict, "april": summary dict, "improvement"}."""
    imps = [e["improvement"] for e in per_seed if e.get("improvement") is not None]
    offp = [e["april"]["mean_offpolicy_fraction"] for e in per_seed if "april" in e]
    return {"seeds": [e["seed"] for e in per_seed], "per_seed": per_seed,
            "mean_improvement": float(np.mean(imps)) if imps else None,
            "std_improvement": float(np.std(imps)) if imps else None,
            "mean_offpolicy_fraction": float(np.mean(offp)) if offp else None,
            "resolved_config": resolved_config}


def write_comparison(out_dir: str, per_seed: list[dict], resolved_config: dict) -> str:
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, "comparison.json")
    with open(path, "w", encoding="utf-8") as f:
        json.dump(comparison_record(per_seed, resolved_config), f, indent=2, sort_keys=True)
        f.write("\n")
    return path
