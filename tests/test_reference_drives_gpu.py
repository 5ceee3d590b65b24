"""The UNMODIFIED reference drives the B200 engine (drop-in proof).

`baseline/_ref` holds the reference package installed from /root/reference/pkg (gitignored; it
travels to the GPU box with the repo snapshot).  Here the reference's own `april_sim.Scheduler`,
`april_sim.rollouts.RolloutSample`, `Simulation` and toy trainer run exactly as shipped; only the
engine object the reference's `build_simulation` picks (src/april_sim/simulate.py:105-121) is
replaced by `paper_2509_18521_b200.LengthDrivenEngine` / `PolicyDrivenEngine`, which the reference
scheduler drives through its 8-member duck type (src/april_sim/scheduler.py:153-171):
  * length-trace replay: canonical step records equal the committed reference goldens;
  * toy policy (the reference's toy_policy_config): every StepReport field the engine determines
    equals the reference's own run (its PolicyDrivenEngine on the CPU, same process), token ids
    included -- the Philox draw, softmax, inverse CDF and STOP rule run on the GPU;
  * convergence parity, the reference's own acceptance criterion (tests/test_acceptance.py:206-225):
    with the B200 engine, final toy rewards of APRIL are within 5 % of the synchronous baseline and
    both exceed 3x the uniform reward, over seeds 0, 1, 2.
"""

import os
import sys

import pytest

import canon
import goldens
import paper_2509_18521_b200 as pb

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "april_sim")):
    pytest.skip("baseline/_ref (the installed reference) is missing: see DESIGN.md §2", allow_module_level=True)
sys.path.insert(0, REF)
import april_sim as a  # noqa: E402
from april_sim import scheduler as ref_scheduler  # noqa: E402
from april_sim import workload as ref_workload  # noqa: E402


def _logging(cls):
    """Event log in the golden generator's format (tests/golden/make_goldens.py)."""

    class Logged(cls):
        def __init__(self, *args, **kw):
            super().__init__(*args, **kw)
            self.event_log = []

        def decode_until_event(self):
            evs = super().decode_until_event()
            for ev in evs:
                s = ev.sample
                self.event_log.append([self.iteration_index, s.instance_id, s.sample_index, ev.tokens, ev.reason])
            return evs

    return Logged


def _ref_dist(d, l_max):
    if d[0] == "constant":
        return ref_workload.LengthDistribution.constant(int(d[1]), l_max)
    return ref_workload.LengthDistribution.lognormal(d[1], d[2], l_max)


@pytest.mark.parametrize("name,model", [("C1", None), ("E_samples", None), ("E_pool", None), ("E_cap", None),
                                        ("C3", None), ("C1", "tiny")])
def test_reference_scheduler_replays_on_gpu_engine(name, model):
    cfg = canon.CONFIGS[name]
    g = goldens.replay(name, "april")
    ecfg = a.EngineConfig(d0=cfg.get("d0", 0.05), d1=cfg.get("d1", 0.002), max_slots=cfg["slots"], l_max=cfg["l_max"])
    kw = {}
    if model:
        kw = dict(model=pb.PRESETS[model], sampling=pb.SamplingConfig(temperature=0.8), prompt_len=64,
                  kv_resume="reprefill", nondeterministic_gemm=True)
    eng = _logging(pb.LengthDrivenEngine)(ecfg, global_seed=cfg["seed"], **kw)
    scfg = ref_scheduler.SchedulerConfig(rollout_batch_size=cfg["n"], samples_per_prompt=cfg["g"],
                                         over_sampling_batch_size=cfg["n_prime"], mode="april",
                                         trigger=cfg.get("trigger", "groups"))
    sampler = ref_workload.LengthSampler(_ref_dist(cfg["dist"], cfg["l_max"]), cfg["rho"], cfg["seed"])
    sched = ref_scheduler.Scheduler(scfg, eng, ref_workload.InstanceSource(group_size=cfg["g"]), sampler)
    assert type(sched).__module__ == "april_sim.scheduler"
    for k, ref in enumerate(g["records"]):
        eng.event_log = []
        out = sched.run_step(k)
        assert type(out.batch[0].samples[0]).__module__ == "april_sim.rollouts"
        rec = canon.step_record(sched, out, eng.event_log)
        ref = {key: v for key, v in ref.items() if key != "rollout_wall_time"}
        assert rec == ref, f"step {k}: " + str(canon.first_diff(rec, ref))
    eng.close()


_ENGINE_FIELDS = ("step", "tokens_generated", "completed_groups", "carried_in_tokens", "offpolicy_fraction",
                  "offpolicy_sample_fraction", "staleness_histogram", "sigma_batch", "sigma_instance", "mean_reward",
                  "buffer_size_after", "train_wall_time")


def _toy_sim(seed, mode, engine, steps):
    cfg = a.toy_policy_config().with_overrides(**{"run.seed": seed, "scheduler.mode": mode, "run.steps": steps})
    sim = a.build_simulation(cfg)
    if engine == "b200":
        sim.scheduler.engine = pb.PolicyDrivenEngine(cfg.engine, global_seed=seed)
    return sim


@pytest.mark.parametrize("mode", ["april", "baseline"])
def test_reference_simulation_with_gpu_engine_equals_reference_run(mode):
    steps = 60
    mine = _toy_sim(4, mode, "b200", steps)
    ref = _toy_sim(4, mode, "reference", steps)
    for k in range(steps):
        r1, r2 = mine.run_step(), ref.run_step()
        d1, d2 = r1.to_json_dict(), r2.to_json_dict()
        for f in _ENGINE_FIELDS:
            assert d1[f] == d2[f], (k, f, d1[f], d2[f])
    # the policies trained on the two runs' batches are identical, bit for bit
    assert list(mine.policy.logits) == list(ref.policy.logits)
    mine.scheduler.engine.close()


def test_convergence_parity_with_gpu_engine():
    """tests/test_acceptance.py:206-225 of the reference with its engine replaced by the B200 engine."""
    uniform = 1.0 / (4 + 1)
    finals = {"baseline": [], "april": []}
    for seed in (0, 1, 2):
        for mode in ("baseline", "april"):
            sim = _toy_sim(seed, mode, "b200", 300)
            sim.run()
            finals[mode].append(sim.reports[-1].mean_reward)
            sim.scheduler.engine.close()
    base = sum(finals["baseline"]) / 3
    apr = sum(finals["april"]) / 3
    assert base > 3 * uniform and apr > 3 * uniform, finals
    assert abs(apr - base) / base <= 0.05, finals


_LENGTH_FIELDS = tuple(f for f in _ENGINE_FIELDS if f != "mean_reward")


def test_build_simulation_runs_reference_config_on_gpu():
    """`pb.build_simulation` (the drop-in for simulate.py:105-121) takes the reference's own
    RunConfig: its default length-driven run (N 32, G 8, N' 64, lognormal tail) replayed on the GPU
    engine gives the reference run's step reports (every field the engine determines), and the
    toy-policy run with the reference trainer's update rule trains the same policy bit for bit."""
    cfg = a.default_config().with_overrides(**{"run.steps": 6, "run.write_manifest": True})
    mine, ref = pb.build_simulation(cfg), a.build_simulation(cfg)
    for k in range(cfg.run.steps):
        d1, d2 = mine.run_step().to_json_dict(), ref.run_step().to_json_dict()
        for f in _LENGTH_FIELDS:
            assert d1[f] == d2[f], (k, f, d1[f], d2[f])
    assert len(mine.manifest) == len(ref.manifest)
    assert [tuple(r.values()) for r in mine.manifest] == [
        (r.step, r.instance_id, r.sample_index, r.start_version, r.complete_version, r.tokens) for r in ref.manifest]
    assert mine.summary().buffer_high_water == ref.summary().buffer_high_water
    mine.close()

    cfg = a.toy_policy_config().with_overrides(**{"run.steps": 25, "run.seed": 3})
    with pytest.raises(pb.ConfigError):
        pb.build_simulation(cfg)  # a policy-driven run needs the trainer's update rule
    mine = pb.run_simulation(cfg, policy_update=a.reinforce_update)
    ref = a.run_simulation(cfg)
    for r1, r2 in zip(mine.reports, ref.reports):
        d1, d2 = r1.to_json_dict(), r2.to_json_dict()
        for f in _ENGINE_FIELDS:
            assert d1[f] == d2[f], (r1.step, f, d1[f], d2[f])
    assert list(mine.policy.logits) == list(ref.policy.logits)
    mine.close()
