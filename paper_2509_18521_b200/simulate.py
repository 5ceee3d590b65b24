"""Whole-run orchestration on the GPU engines: the drop-in for src/april_sim/simulate.py:34-127.

`build_simulation(config)` is the place where the reference picks its engine
(simulate.py:105-121); here it builds the B200 engine of the same workload mode behind the same
`Scheduler`, so a run configured with the reference's `RunConfig` executes on the GPU.  Any object
with its five sections works (workload: distribution / parameters / correlate_within_group / mode;
engine; scheduler; train; run); the config classes, JSON round trip and presets themselves stay the
reference's (`config.py`: configuration plumbing, out of scope per SURVEY.md section 2).

Policy-driven runs update the toy policy between steps with the reference trainer's rule, which is
not on the rollout path: pass it as `policy_update(policy, samples,
advantages, train_config) -> PolicyParams` (e.g. `april_sim.reinforce_update`).  Rewards and the
group-relative advantages are this package's (`reward`, K6 `group_advantages`).
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field
from typing import Any, Callable

from . import metrics
from .engine import EngineConfig, LengthDrivenEngine, PolicyDrivenEngine
from .errors import ConfigError
from .policy import PolicyParams, group_advantages, reward
from .scheduler import Scheduler, SchedulerConfig
from .workload import InstanceSource, LengthDistribution, LengthSampler, load_histogram_csv

POLICY_DRIVEN = "policy_driven"  # config.py:19-20
LENGTH_DRIVEN = "length_driven"


def _section(obj, cls):
    """The reference's section dataclass (or a dict) as this package's own config class."""
    if isinstance(obj, cls):
        return obj
    vals = dataclasses.asdict(obj) if dataclasses.is_dataclass(obj) else dict(obj)
    return cls(**{f.name: vals[f.name] for f in dataclasses.fields(cls) if f.name in vals})


def length_distribution(workload, l_max: int) -> LengthDistribution:
    """The trace's length law from a workload section (config.py:36-58 names and parameters)."""
    name, p = workload.distribution, dict(workload.parameters)
    makers = {
        "constant": lambda: LengthDistribution.constant(int(p["value"]), l_max),
        "geometric": lambda: LengthDistribution.geometric(float(p["p_stop"]), l_max),
        "lognormal": lambda: LengthDistribution.lognormal(float(p["mu_ln"]), float(p["sigma_ln"]), l_max),
        "pareto": lambda: LengthDistribution.pareto(float(p["alpha"]), float(p["x_min"]), l_max),
        "empirical": lambda: load_histogram_csv(str(p["path"]), l_max=l_max),
    }
    if name not in makers:
        raise ConfigError(f"workload.distribution: unknown distribution {name!r}")
    try:
        return makers[name]()
    except KeyError as exc:
        raise ConfigError(f"workload.parameters: missing {exc.args[0]!r}") from exc


@dataclass
class Simulation:
    """One run: a scheduler over a GPU engine, the toy policy (policy-driven mode) and the per-step
    reports, manifest rows and event records (simulate.py:34-100)."""

    config: Any
    scheduler: Scheduler
    policy: PolicyParams | None
    policy_update: Callable | None = None
    reports: list = field(default_factory=list)
    manifest: list = field(default_factory=list)
    events: list = field(default_factory=list)
    _step: int = 0

    @property
    def policy_driven(self) -> bool:
        return self.config.workload.mode == POLICY_DRIVEN

    def run_step(self) -> metrics.StepReport:
        k = self._step
        outcome = self.scheduler.run_step(k, self.policy)
        samples = outcome.batch_samples()
        mean_reward = 0.0
        if self.policy_driven:
            tr = self.config.train
            rewards = [reward(s, tr.target_token) for s in samples]
            mean_reward = sum(rewards) / len(rewards) if rewards else 0.0
            adv, at = [], 0
            for g in outcome.batch:  # groups in batch order, each normalised on its own
                n = len(g.samples)
                adv.extend(group_advantages(rewards[at:at + n], tr.advantage_mode, tr.std_eps))
                at += n
            self.policy = self.policy_update(self.policy, samples, adv, tr)
        tokens = sum(s.total_tokens for s in samples)
        train = self.config.train
        rep = metrics.build_step_report(outcome, peak_rate=self.config.engine.peak_rate,
                                        train_wall_time=train.c0 + train.c1 * tokens,  # policy.py:201-203
                                        mean_reward=mean_reward)
        self.reports.append(rep)
        if self.config.run.write_manifest:
            self.manifest.extend(dict(step=k, instance_id=s.instance_id, sample_index=s.sample_index,
                                      start_version=s.start_version, complete_version=s.complete_version,
                                      tokens=s.total_tokens) for g in outcome.batch for s in g.samples)
        self._step += 1
        return rep

    def run(self) -> list:
        for _ in range(self.config.run.steps):
            self.run_step()
        return self.reports

    def summary(self, baseline=None) -> metrics.RunSummary:
        return metrics.summarize_run(self.reports, baseline, buffer_high_water=self.scheduler.buffer.high_water)

    def close(self) -> None:
        self.scheduler.engine.close()


def build_simulation(config, policy_update: Callable | None = None, **engine_kw) -> Simulation:
    """The GPU engine for `config`'s workload mode behind the Scheduler (simulate.py:105-121).
    `engine_kw` goes to the engine (e.g. model=PRESETS[...] for the transformer decoder)."""
    seed = config.run.seed
    ecfg = _section(config.engine, EngineConfig)
    scfg = _section(config.scheduler, SchedulerConfig)
    source = InstanceSource(group_size=scfg.samples_per_prompt)
    mode = config.workload.mode
    if mode == POLICY_DRIVEN:
        if policy_update is None:
            raise ConfigError("a policy-driven run needs policy_update (the toy trainer's update rule)")
        engine = PolicyDrivenEngine(ecfg, global_seed=seed, **engine_kw)
        sampler, policy = None, PolicyParams.uniform(config.train.vocab_size)
    elif mode == LENGTH_DRIVEN:
        engine = LengthDrivenEngine(ecfg, **engine_kw)
        sampler = LengthSampler(length_distribution(config.workload, ecfg.l_max),
                                config.workload.correlate_within_group, seed)
        policy = None
    else:
        raise ConfigError(f"workload.mode: unknown mode {mode!r}")
    sim = Simulation(config=config, scheduler=Scheduler(scfg, engine, source, sampler), policy=policy,
                     policy_update=policy_update)
    if config.run.write_events:
        sim.scheduler.event_sink = sim.events
    return sim


def run_simulation(config, policy_update: Callable | None = None, **engine_kw) -> Simulation:
    sim = build_simulation(config, policy_update, **engine_kw)
    sim.run()
    return sim
