"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_goldens.py [/root/reference/pkg/src]

Outputs (committed, they travel to the GPU box; nothing at test time reads
/root/reference):
  tests/golden/replay_<cfg>_<mode>.json.gz   full per-step records (tests/canon.py)
  tests/golden/replay_digests.json           sha256 per step, for every config
  tests/golden/toy_<mode>.json.gz            toy policy-driven run (seed 4, 60 steps):
                                             per-step records incl. token ids and
                                             behaviour logprobs, plus StepReports
  tests/golden/philox.json                   raw Philox words / draws for a few keys

The toy run reproduces the reference's own fixtures
(frontend/tests/fixtures/sample_run|sample_baseline/steps.jsonl); this script
asserts that before writing anything.
"""

from __future__ import annotations

import gzip
import json
import math
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/ for canon

import canon  # noqa: E402

REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402
from april_sim import engine as ref_engine  # noqa: E402
from april_sim import metrics as ref_metrics  # noqa: E402
from april_sim import policy as ref_policy  # noqa: E402
from april_sim.rng import LANE_POLICY_TOKENS, Stream, philox_key  # noqa: E402
from april_sim.scheduler import Scheduler, SchedulerConfig  # noqa: E402
from april_sim.workload import InstanceSource, LengthDistribution, LengthSampler  # noqa: E402


def _logging(cls):
    class Logged(cls):
        def __init__(self, *a, **k):
            super().__init__(*a, **k)
            self.event_log = []

        def decode_until_event(self):
            evs = super().decode_until_event()
            for ev in evs:
                s = ev.sample
                self.event_log.append([self.iteration_index, s.instance_id, s.sample_index, ev.tokens, ev.reason])
            return evs

    return Logged


LenEngine = _logging(ref_engine.LengthDrivenEngine)
PolEngine = _logging(ref_engine.PolicyDrivenEngine)


def _dist(d, l_max):
    kind = d[0]
    if kind == "constant":
        return LengthDistribution.constant(int(d[1]), l_max)
    if kind == "lognormal":
        return LengthDistribution.lognormal(d[1], d[2], l_max)
    raise ValueError(kind)


def run_replay(cfg, mode, steps):
    ecfg = ref_engine.EngineConfig(d0=cfg.get("d0", 0.05), d1=cfg.get("d1", 0.002), max_slots=cfg["slots"],
                                   l_max=cfg["l_max"])
    eng = LenEngine(ecfg)
    scfg = SchedulerConfig(rollout_batch_size=cfg["n"], samples_per_prompt=cfg["g"],
                           over_sampling_batch_size=cfg["n_prime"], mode=mode,
                           trigger=cfg.get("trigger", "groups"))
    sampler = LengthSampler(_dist(cfg["dist"], cfg["l_max"]), cfg["rho"], cfg["seed"])
    sched = Scheduler(scfg, eng, InstanceSource(group_size=cfg["g"]), sampler)
    recs = []
    for k in range(steps):
        eng.event_log = []
        out = sched.run_step(k)
        rec = canon.step_record(sched, out, eng.event_log)
        rec["rollout_wall_time"] = out.rollout_wall_time
        recs.append(rec)
    return recs


def run_toy(mode):
    t = canon.TOY
    ecfg = ref_engine.EngineConfig(d0=t["d0"], d1=t["d1"], max_slots=t["slots"], l_max=t["l_max"])
    eng = PolEngine(ecfg, global_seed=t["seed"])
    scfg = SchedulerConfig(rollout_batch_size=t["n"], samples_per_prompt=t["g"],
                           over_sampling_batch_size=t["n_prime"], mode=mode)
    sched = Scheduler(scfg, eng, InstanceSource(group_size=t["g"]), None)
    tcfg = ref_policy.TrainConfig(vocab_size=t["vocab"], target_token=t["target"], learning_rate=t["lr"])
    params = ref_policy.PolicyParams.uniform(t["vocab"])
    recs, reports = [], []
    for k in range(t["steps"]):
        eng.event_log = []
        logits_in = [float(x) for x in params.logits]
        out = sched.run_step(k, params)
        samples = out.batch_samples()
        rewards = [ref_policy.reward(s, t["target"]) for s in samples]
        adv = []
        pos = 0
        for g in out.batch:
            adv.extend(ref_policy.group_advantages(rewards[pos:pos + len(g.samples)], tcfg.advantage_mode,
                                                   tcfg.std_eps))
            pos += len(g.samples)
        rec = canon.step_record(sched, out, eng.event_log, with_tokens=True)
        rec["logits_in"] = logits_in
        rec["rewards"] = rewards
        rec["advantages"] = [float(a) for a in adv]
        params = ref_policy.reinforce_update(params, samples, adv, tcfg)
        mean_reward = 0.0
        for r in rewards:  # naive left-to-right, as the fixtures were produced
            mean_reward += r
        mean_reward /= len(rewards)
        batch_tokens = sum(s.total_tokens for s in samples)
        rep = ref_metrics.build_step_report(out, peak_rate=ecfg.peak_rate,
                                            train_wall_time=ref_policy.train_wall_time(batch_tokens, tcfg),
                                            mean_reward=mean_reward)
        rec["rollout_wall_time"] = out.rollout_wall_time
        recs.append(rec)
        reports.append(rep.to_json_dict())
    return recs, reports


def check_fixture(reports, path):
    if not os.path.exists(path):
        print(f"  (fixture {path} absent; skipped)")
        return
    with open(path) as f:
        fx = [json.loads(line) for line in f]
    assert len(fx) == len(reports), (len(fx), len(reports))
    for a, b in zip(reports, fx):
        for k in b:
            if k == "mean_reward":
                assert math.isclose(a[k], b[k], rel_tol=0, abs_tol=1e-15), (k, a[k], b[k])
            else:
                assert a[k] == b[k], (a["step"], k, a[k], b[k])
    print(f"  reproduces {path} ({len(fx)} steps)")


def _dump(name, obj):
    with gzip.open(os.path.join(HERE, name), "wt") as f:
        json.dump(obj, f, separators=(",", ":"))


def main():
    digests = {}
    for name, cfg in canon.CONFIGS.items():
        for mode in ("april", "baseline"):
            steps = cfg["steps"] if mode == "april" else canon.SYNC_STEPS.get(name, 0)
            if not steps:
                continue
            recs = run_replay(cfg, mode, steps)
            digests[f"{name}/{mode}"] = [canon.digest({k: v for k, v in r.items() if k != "rollout_wall_time"})
                                         for r in recs]
            size = len(json.dumps(recs))
            if size < 3_000_000:
                _dump(f"replay_{name}_{mode}.json.gz", {"config": cfg, "mode": mode, "records": recs})
            print(f"{name}/{mode}: {steps} steps, {size/1e6:.2f} MB records, "
                  f"iters={recs[-1]['iteration_index']} tokens={recs[-1]['cumulative_tokens']}")
    with open(os.path.join(HERE, "replay_digests.json"), "w") as f:
        json.dump(digests, f, indent=1)

    fx_root = os.path.join(os.path.dirname(REF), "frontend", "tests", "fixtures")
    for mode, fx in (("april", "sample_run"), ("baseline", "sample_baseline")):
        recs, reports = run_toy(mode)
        check_fixture(reports, os.path.join(fx_root, fx, "steps.jsonl"))
        _dump(f"toy_{mode}.json.gz", {"config": canon.TOY, "mode": mode, "records": recs, "reports": reports})
        print(f"toy/{mode}: done")

    # raw Philox words for a few keys (pins the counter/key convention absolutely)
    ph = []
    for (seed, lane, iid, sidx) in [(0, 2, 0, 0), (4, 2, 17, 3), (123456789, 0, 99, 7), (-5, 1, 2**40, 0)]:
        key = philox_key(seed, lane, iid, sidx)
        gen = Stream(seed, lane, iid, sidx).generator(0)
        draws = [float(x) for x in gen.random(9)]
        gen5 = Stream(seed, lane, iid, sidx).generator(5)
        ph.append({"addr": [seed, lane, iid, sidx], "key": str(key), "draws0": draws,
                   "draws5": [float(x) for x in gen5.random(4)]})
    with open(os.path.join(HERE, "philox.json"), "w") as f:
        json.dump(ph, f, indent=1)

    # trace lengths for the sampler (ndtri path) at a few addresses
    tl = []
    for name in ("C1", "C2", "C3", "C4_3", "C5"):
        cfg = canon.CONFIGS[name]
        smp = LengthSampler(_dist(cfg["dist"], cfg["l_max"]), cfg["rho"], cfg["seed"])
        tl.append({"config": name, "lengths": [[i, j, smp.target_length(i, j)] for i in range(0, 200, 7)
                                               for j in range(cfg["g"])]})
    with open(os.path.join(HERE, "trace_lengths.json"), "w") as f:
        json.dump(tl, f)
    _ = LANE_POLICY_TOKENS, np
    print("goldens written")


if __name__ == "__main__":
    main()
