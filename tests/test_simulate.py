"""Host side of the run orchestration drop-in (paper_2509_18521_b200/simulate.py): the reference's
RunConfig sections map onto this package's config classes and length laws exactly (no GPU)."""

import dataclasses
import os
import sys

import pytest

import paper_2509_18521_b200 as pb
from paper_2509_18521_b200 import simulate

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "april_sim")):
    pytest.skip("baseline/_ref (the installed reference) is missing: see DESIGN.md §2", allow_module_level=True)
sys.path.insert(0, REF)
import april_sim as a  # noqa: E402
from april_sim.config import WorkloadConfig  # noqa: E402


@pytest.mark.parametrize("dist,params", [("lognormal", {"mu_ln": 6.6, "sigma_ln": 1.0}),
                                         ("constant", {"value": 37}), ("geometric", {"p_stop": 0.01}),
                                         ("pareto", {"alpha": 1.3, "x_min": 40.0})])
def test_length_law_from_reference_workload_section(dist, params):
    wl = WorkloadConfig(distribution=dist, parameters=params)
    mine = simulate.length_distribution(wl, 4096)
    ref = wl.build_distribution(4096)
    assert dataclasses.asdict(mine) == dataclasses.asdict(ref)


def test_config_sections_convert():
    cfg = a.toy_policy_config()
    e = simulate._section(cfg.engine, pb.EngineConfig)
    s = simulate._section(cfg.scheduler, pb.SchedulerConfig)
    assert dataclasses.asdict(e) == dataclasses.asdict(cfg.engine)
    assert dataclasses.asdict(s) == dataclasses.asdict(cfg.scheduler)
    assert e.peak_rate == cfg.engine.peak_rate


def test_bad_workload_names_raise_config_error():
    with pytest.raises(pb.ConfigError):
        simulate.length_distribution(WorkloadConfig(distribution="lognormal", parameters={"mu_ln": 1.0}), 64)
    bad = dataclasses.replace(WorkloadConfig(), distribution="zipf")
    with pytest.raises(pb.ConfigError):
        simulate.length_distribution(bad, 64)
