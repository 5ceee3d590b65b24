"""Run outputs in the reference's schema (cli.py:50-74, 117-129)."""

import json
import os

import numpy as np

import paper_2509_18521_b200 as pb
from paper_2509_18521_b200 import report
from paper_2509_18521_b200.metrics import StepReport

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "output_schema.json")


def _gold():
    with open(GOLD) as f:
        return json.load(f)


def test_step_records_round_trip_byte_identical(tmp_path):
    g = _gold()
    reports = [StepReport.from_json_dict(d) for d in g["steps"]]
    summary = pb.summarize_run(reports, buffer_high_water=64)
    report.write_run_outputs(str(tmp_path), reports, summary, {"engine": {}, "run": {}, "scheduler": {},
                                                                 "train": {}, "workload": {}})
    lines = (tmp_path / "steps.jsonl").read_text().splitlines()
    assert lines == g["steps_raw_lines"]
    s = json.loads((tmp_path / "summary.json").read_text())
    assert sorted(s.keys()) == g["summary_keys"]
    assert sorted(s["resolved_config"].keys()) == g["resolved_config_sections"]
    assert s["steps"] == 5 and s["total_tokens"] == sum(d["tokens_generated"] for d in g["steps"])


def test_manifest_events_and_comparison(tmp_path):
    g = _gold()
    reports = [StepReport.from_json_dict(d) for d in g["steps"]]
    base = [StepReport.from_json_dict(dict(d, throughput=d["throughput"] / 2)) for d in g["steps"]]
    summ_a = pb.summarize_run(reports, baseline=base)
    summ_b = pb.summarize_run(base)
    rows = [(0, 3, 1, 0, 0, 17), (1, 4, 0, 0, 1, 250)]
    report.write_run_outputs(str(tmp_path / "april"), reports, summ_a, {}, manifest=rows,
                             events=[{"clock": 0.5, "sample_id": "3-1", "tokens": 17, "reason": "stop_token",
                                      "iteration_index": 4}])
    text = (tmp_path / "april" / "samples.csv").read_text().splitlines()
    assert text[0] == "step,instance_id,sample_index,start_version,complete_version,tokens"
    assert text[1:] == ["0,3,1,0,0,17", "1,4,0,0,1,250"]
    assert json.loads((tmp_path / "april" / "events.jsonl").read_text())["tokens"] == 17
    per_seed = [{"seed": 0, "baseline": summ_b.to_json_dict(), "april": summ_a.to_json_dict(),
                 "improvement": summ_a.relative_throughput_improvement}]
    path = report.write_comparison(str(tmp_path), per_seed, {})
    c = json.load(open(path))
    assert sorted(c.keys()) == ["mean_improvement", "mean_offpolicy_fraction", "per_seed", "resolved_config",
                                "seeds", "std_improvement"]
    np.testing.assert_allclose(c["mean_improvement"], 1.0)
