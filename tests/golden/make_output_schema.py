"""Freeze a few records of the reference's run-output fixtures (pkg/frontend/tests/fixtures/sample_run:
steps.jsonl, summary.json) as tests/golden/output_schema.json, so the writer in
paper_2509_18521_b200/report.py is checked against the reference's on-disk schema without
/root/reference at test time.  Run here (the reference tree exists only in this container):

    python tests/golden/make_output_schema.py
"""
import json
import os

SRC = "/root/reference/pkg/frontend/tests/fixtures/sample_run"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "output_schema.json")


def main():
    with open(os.path.join(SRC, "steps.jsonl")) as f:
        steps = [json.loads(line) for line in f][:5]
    with open(os.path.join(SRC, "summary.json")) as f:
        summary = json.load(f)
    with open(os.path.join(SRC, "steps.jsonl")) as f:
        raw = [line.rstrip("\n") for line in f][:5]
    out = {"source": "pkg/frontend/tests/fixtures/sample_run (reference run output, toy policy, seed 4)",
           "steps": steps, "steps_raw_lines": raw, "summary_keys": sorted(summary.keys()),
           "resolved_config_sections": sorted(summary["resolved_config"].keys())}
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
