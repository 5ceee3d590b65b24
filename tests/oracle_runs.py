"""Drivers that run the CPU oracle over the canonical configs (test helpers)."""

from __future__ import annotations

import canon
from oracle import sim_ref


def oracle_replay(cfg: dict, mode: str, steps: int):
    c = dict(cfg, mode=mode)
    eng, sch = sim_ref.make_oracle(c)
    recs = []
    for k in range(steps):
        eng.event_log = []
        out = sch.run_step(k)
        rec = canon.step_record(sch, out, eng.event_log)
        recs.append(rec)
    return recs


def oracle_toy(mode: str, steps: int | None = None):
    t = canon.TOY
    eng = sim_ref.OracleEngine(t["d0"], t["d1"], t["slots"], t["l_max"], mode="policy", seed=t["seed"])
    sch = sim_ref.OracleScheduler(t["n"], t["g"], t["n_prime"], eng, mode=mode)
    import numpy as np

    z = np.zeros(t["vocab"] + 1)
    recs = []
    for k in range(steps or t["steps"]):
        eng.event_log = []
        out = sch.run_step(k, z)
        samples = out.batch_samples()
        rewards = [sim_ref.reward_of(s, t["target"]) for s in samples]
        adv = []
        pos = 0
        for g in out.batch:
            adv.extend(sim_ref.advantages_of(rewards[pos:pos + len(g.samples)]))
            pos += len(g.samples)
        rec = canon.step_record(sch, out, eng.event_log, with_tokens=True)
        rec["logits_in"] = [float(x) for x in z]
        rec["rewards"] = rewards
        rec["advantages"] = [float(a) for a in adv]
        z = sim_ref.reinforce_step(z, samples, adv, t["lr"])
        recs.append(rec)
    return recs
