"""Drivers that run the B200 product over the canonical configs (test helpers)."""

from __future__ import annotations

import numpy as np

import canon
import paper_2509_18521_b200 as pb


def _dist(cfg):
    d = cfg["dist"]
    if d[0] == "constant":
        return pb.LengthDistribution.constant(int(d[1]), cfg["l_max"])
    return pb.LengthDistribution.lognormal(d[1], d[2], cfg["l_max"])


def make_scheduler(cfg: dict, mode: str, fused: bool = True, engine=None, model=None, sampling=None, **ekw):
    ecfg = pb.EngineConfig(d0=cfg.get("d0", 0.05), d1=cfg.get("d1", 0.002), max_slots=cfg["slots"],
                           l_max=cfg["l_max"])
    eng = engine or pb.LengthDrivenEngine(ecfg, global_seed=cfg.get("seed", 0), model=model, sampling=sampling,
                                          **ekw)
    scfg = pb.SchedulerConfig(rollout_batch_size=cfg["n"], samples_per_prompt=cfg["g"],
                              over_sampling_batch_size=cfg["n_prime"], mode=mode,
                              trigger=cfg.get("trigger", "groups"))
    sampler = pb.LengthSampler(_dist(cfg), cfg["rho"], cfg["seed"])
    sched = pb.Scheduler(scfg, eng, pb.InstanceSource(group_size=cfg["g"]), sampler)
    sched._fused = fused
    sched.event_sink = []
    return sched


def step_events(sched):
    evs = [[r["iteration_index"], *map(int, r["sample_id"].split(":")), r["tokens"], r["reason"]]
           for r in sched.event_sink if r["reason"] != "aborted"]
    sched.event_sink.clear()
    return evs


def product_replay(cfg: dict, mode: str, steps: int, fused: bool = True, **kw):
    sched = make_scheduler(cfg, mode, fused=fused, **kw)
    recs = []
    for k in range(steps):
        out = sched.run_step(k)
        recs.append(canon.step_record(sched, out, step_events(sched)))
    return recs, sched


def product_toy(mode: str, golden_records, steps: int, fused: bool = True):
    t = canon.TOY
    ecfg = pb.EngineConfig(d0=t["d0"], d1=t["d1"], max_slots=t["slots"], l_max=t["l_max"])
    eng = pb.PolicyDrivenEngine(ecfg, global_seed=t["seed"])
    scfg = pb.SchedulerConfig(rollout_batch_size=t["n"], samples_per_prompt=t["g"],
                              over_sampling_batch_size=t["n_prime"], mode=mode)
    sched = pb.Scheduler(scfg, eng, pb.InstanceSource(group_size=t["g"]), None)
    sched._fused = fused
    sched.event_sink = []
    recs = []
    for k in range(steps):
        z = np.asarray(golden_records[k]["logits_in"], dtype=float)  # teacher-forced policy
        out = sched.run_step(k, pb.PolicyParams(z, k))
        samples = out.batch_samples()
        rewards = [pb.reward(s, t["target"]) for s in samples]
        adv = pb.batch_advantages(rewards, t["g"], "mean_baseline")
        rec = canon.step_record(sched, out, step_events(sched), with_tokens=True)
        rec["logits_in"] = [float(x) for x in z]
        rec["rewards"] = rewards
        rec["advantages"] = [float(a) for a in adv]
        recs.append(rec)
    return recs
