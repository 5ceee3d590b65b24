"""CPU restatement of the reference rollout path — TEST INFRASTRUCTURE ONLY.

Restates, in one module, the semantics of
  * the trace source     src/april_sim/workload.py:126-148, 229-235
  * the decode engine    src/april_sim/engine.py:98-289
  * the buffer/scheduler src/april_sim/scheduler.py:59-393
  * sampling/reward/advantages src/april_sim/policy.py:87-124
so that tests (and the CPU-baseline leg of bench.py) can replay any
configuration without the reference installed.  It is checked against the
reference-generated goldens in tests/golden/ (see tests/test_oracle.py).

Everything is event-exact: iteration_index / cumulative_tokens follow
engine.py:167-171, event order follows the stable slot filter
(engine.py:174-179), and the scheduler's bookkeeping follows
scheduler.py:232-318 step for step.  Simulated clock is kept too
(d0 + d1*b per iteration) so the oracle's StepOutcome matches the
reference's field for field.
"""

from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field

import numpy as np
from scipy.special import ndtr, ndtri

from . import rng_ref

PENDING, ACTIVE, PAUSED, COMPLETED = "pending", "active", "paused", "completed"
STOP_TOKEN, TARGET_LENGTH, MAX_LENGTH = "stop_token", "target_length", "max_length"


class OracleContract(RuntimeError):
    pass


# --------------------------------------------------------------------------
# trace source (workload.py:126-148, 229-235)
# --------------------------------------------------------------------------


def _clip_u(u):
    return np.clip(np.asarray(u, dtype=float), 2.0 ** -53, 1.0 - 2.0 ** -53)


@dataclass(frozen=True)
class TraceDist:
    kind: str  # constant | lognormal | geometric | pareto
    l_max: int
    a: float = 0.0  # value | mu_ln | p_stop | alpha
    b: float = 0.0  # -     | sigma | -      | x_min

    def length(self, u: float) -> int:
        uu = _clip_u(u)
        if self.kind == "constant":
            raw = np.full_like(uu, float(self.a))
        elif self.kind == "lognormal":
            raw = np.floor(np.exp(self.a + self.b * ndtri(uu)) + 0.5)
        elif self.kind == "geometric":
            raw = np.ones_like(uu) if self.a >= 1.0 else np.ceil(np.log1p(-uu) / math.log1p(-self.a))
        elif self.kind == "pareto":
            raw = np.floor(self.b * np.power(1.0 - uu, -1.0 / self.a) + 0.5)
        else:
            raise ValueError(self.kind)
        return int(np.clip(raw, 1, self.l_max).astype(np.int64)[()])


def trace_length(dist: TraceDist, rho: float, seed: int, iid: int, sidx: int) -> int:
    """Gaussian-copula target length (workload.py:229-235)."""
    z = float(ndtri(rng_ref.clamped_uniform(rng_ref.stream_key(seed, rng_ref.LANE_SAMPLE_LENGTH, iid, sidx), 0)))
    if rho > 0.0:
        zs = float(ndtri(rng_ref.clamped_uniform(rng_ref.stream_key(seed, rng_ref.LANE_INSTANCE_SHARED, iid, 0), 0)))
        z = rho * zs + math.sqrt(1.0 - rho * rho) * z
    return dist.length(float(ndtr(z)))


# --------------------------------------------------------------------------
# samples / groups (rollouts.py:27-128)
# --------------------------------------------------------------------------


@dataclass
class OSeg:
    version: int
    token_count: int = 0
    tokens: list | None = None
    behavior_logprobs: list | None = None


@dataclass
class OSample:
    instance_id: int
    sample_index: int
    status: str = PENDING
    segments: list = field(default_factory=list)
    target_length: int | None = None
    start_version: int | None = None
    complete_version: int | None = None
    finish_reason: str | None = None
    paused_at: tuple | None = None

    @property
    def total_tokens(self) -> int:
        return sum(s.token_count for s in self.segments)

    @property
    def sample_id(self) -> str:
        return f"{self.instance_id}:{self.sample_index}"

    def token_ids(self):
        out = []
        for s in self.segments:
            out.extend(s.tokens)
        return out

    def behavior_logprob_trace(self):
        out = []
        for s in self.segments:
            out.extend(s.behavior_logprobs)
        return out


@dataclass
class OGroup:
    instance_id: int
    samples: list
    completed_count: int = 0
    completion_seq: tuple | None = None

    @property
    def complete(self) -> bool:
        return self.completed_count == len(self.samples)

    def total_tokens(self) -> int:
        return sum(s.total_tokens for s in self.samples)


# --------------------------------------------------------------------------
# engine (engine.py:98-289)
# --------------------------------------------------------------------------


class OracleEngine:
    """mode "length": stop at min(target, l_max); mode "policy": toy softmax."""

    def __init__(self, d0, d1, max_slots, l_max, mode="length", seed=0):
        self.d0, self.d1, self.S, self.l_max = d0, d1, max_slots, l_max
        self.mode, self.seed = mode, seed
        self.clock = 0.0
        self.iteration_index = 0
        self.cumulative_tokens = 0
        self.version = 0
        self.slots: list[list] = []  # [sample, remaining, stop_at, cursor]
        self._queue: deque = deque()
        self.cdf = self.logp = None
        self.stop_index = -1
        self.event_log: list = []  # [iteration, iid, sidx, tokens, reason]

    @property
    def idle(self):
        return not self.slots and not self._queue

    def begin_step(self, version, params=None):
        if not self.idle:
            raise OracleContract("begin_step requires idle engine")
        self.version = version
        if self.mode == "policy":
            z = np.asarray(params, dtype=float)
            e = np.exp(z - np.max(z))
            p = e / e.sum()
            self.cdf, self.logp, self.stop_index = np.cumsum(p), np.log(p), z.size - 1

    def submit(self, s):
        if s.status not in (PENDING, PAUSED):
            raise OracleContract(f"bad submit status {s.status}")
        self._queue.append(s)

    def _admit(self):
        while self._queue and len(self.slots) < self.S:
            s = self._queue.popleft()
            s.status = ACTIVE
            if s.segments and s.segments[-1].version >= self.version:
                raise OracleContract("segment versions must strictly increase")
            rec = self.mode == "policy"
            s.segments.append(OSeg(self.version, 0, [] if rec else None, [] if rec else None))
            if s.start_version is None:
                s.start_version = self.version
            if self.mode == "length":
                stop = min(s.target_length, self.l_max)
                rem = stop - s.total_tokens
                if rem <= 0:
                    raise OracleContract("sample already at stop")
                self.slots.append([s, rem, stop, None])
            else:
                key = rng_ref.stream_key(self.seed, rng_ref.LANE_POLICY_TOKENS, s.instance_id, s.sample_index)
                self.slots.append([s, 0, 0, rng_ref.StreamCursor(key, s.total_tokens)])

    def _advance(self, k):
        b = len(self.slots)
        self.clock += k * (self.d0 + self.d1 * b)
        self.iteration_index += k
        self.cumulative_tokens += k * b
        done = []
        for slot in self.slots:
            s = slot[0]
            seg = s.segments[-1]
            if self.mode == "length":
                seg.token_count += k
                slot[1] -= k
                if slot[1] == 0:
                    done.append((slot, MAX_LENGTH if slot[2] >= self.l_max else TARGET_LENGTH))
            else:
                u = slot[3].next_raw()
                tok = min(int(np.searchsorted(self.cdf, u, side="right")), self.stop_index)
                seg.tokens.append(tok)
                seg.behavior_logprobs.append(float(self.logp[tok]))
                seg.token_count += 1
                if tok == self.stop_index:
                    done.append((slot, STOP_TOKEN))
                elif s.total_tokens >= self.l_max:
                    done.append((slot, MAX_LENGTH))
        events = []
        if done:
            gone = {id(sl) for sl, _ in done}
            self.slots = [sl for sl in self.slots if id(sl) not in gone]
            for sl, why in done:
                s = sl[0]
                s.status, s.complete_version, s.finish_reason = COMPLETED, self.version, why
                events.append((s, why))
                self.event_log.append([self.iteration_index, s.instance_id, s.sample_index, s.total_tokens, why])
        return events

    def decode_iteration(self):
        self._admit()
        return self._advance(1) if self.slots else []

    def decode_until_event(self):
        while True:
            self._admit()
            if not self.slots:
                return []
            k = 1 if self.mode == "policy" else max(1, min(sl[1] for sl in self.slots))
            ev = self._advance(k)
            if ev:
                return ev

    def abort_active(self):
        out = []
        for sl in self.slots:
            sl[0].status = PAUSED
            out.append(sl[0])
        self.slots = []
        out.extend(self._queue)
        self._queue.clear()
        return out


# --------------------------------------------------------------------------
# buffer + scheduler (scheduler.py:59-393)
# --------------------------------------------------------------------------


def trigger_fired(n, g, trigger, cg, cs):
    """scheduler.py:59-64."""
    if trigger == "groups":
        return cg >= n
    return cs >= n * g and cg >= n


class OracleBuffer:
    def __init__(self):
        self.parts: list = []
        self.orph: dict = {}
        self.ready: list = []
        self.high_water = 0

    def _hw(self):
        self.high_water = max(self.high_water, self.sample_count())

    def sample_count(self):
        return len(self.parts) + sum(map(len, self.orph.values())) + sum(len(g.samples) for g in self.ready)

    def sample_ids(self):
        ids = [s.sample_id for s in self.parts]
        for lst in self.orph.values():
            ids += [s.sample_id for s in lst]
        for g in self.ready:
            ids += [s.sample_id for s in g.samples]
        return ids

    def partials(self):
        return list(self.parts)


@dataclass
class OOutcome:
    step: int
    batch: list
    rollout_wall_time: float
    tokens_generated: int
    carried_in_tokens: int
    groups_completed: int
    buffer_size_after: int
    pool_size_after: int
    open_group_count: int
    admission_log: list

    def batch_samples(self):
        return [s for g in self.batch for s in g.samples]


class OracleScheduler:
    def __init__(self, n, g, n_prime, engine: OracleEngine, mode="april", trigger="groups",
                 dist: TraceDist | None = None, rho=0.0, seed=0):
        self.n, self.g, self.n_prime = n, g, n_prime
        self.mode, self.trigger = mode, trigger
        self.engine = engine
        self.dist, self.rho, self.seed = dist, rho, seed
        self.buffer = OracleBuffer()
        self.pending_pool: list = []
        self.carry: dict = {}
        self.next_iid = 0
        self.created_samples = 0

    def _new_group(self):
        iid = self.next_iid
        self.next_iid += 1
        ss = []
        for j in range(self.g):
            s = OSample(iid, j)
            if self.dist is not None:
                s.target_length = trace_length(self.dist, self.rho, self.seed, iid, j)
            ss.append(s)
        self.created_samples += self.g
        return OGroup(iid, ss)

    def run_step(self, version, params=None):
        return self._sync(version, params) if self.mode == "baseline" else self._april(version, params)

    def _complete(self, grp):
        grp.completed_count += 1
        if grp.complete:
            grp.completion_seq = (self.engine.iteration_index, grp.instance_id)

    def _sync(self, version, params):
        eng = self.engine
        eng.begin_step(version, params)
        c0, t0 = eng.clock, eng.cumulative_tokens
        groups = [self._new_group() for _ in range(self.n)]
        idx = {gr.instance_id: gr for gr in groups}
        log = []
        for gr in groups:
            for s in gr.samples:
                eng.submit(s)
                log.append(("fresh", s.sample_id))
        while True:
            evs = eng.decode_until_event()
            if not evs:
                break
            for s, _ in evs:
                self._complete(idx[s.instance_id])
        return OOutcome(version, sorted(groups, key=lambda x: x.completion_seq), eng.clock - c0,
                        eng.cumulative_tokens - t0, 0, self.n, 0, 0, self.n, log)

    def _april(self, version, params):
        eng = self.engine
        eng.begin_step(version, params)
        c0, t0 = eng.clock, eng.cumulative_tokens
        opened: dict = {}
        carried = cg = cs = this_step = 0
        for gr in sorted(self.buffer.ready, key=lambda x: x.completion_seq):
            opened[gr.instance_id] = gr
            cg += 1
            cs += len(gr.samples)
            carried += gr.total_tokens()
        self.buffer.ready = []
        log = []
        if not trigger_fired(self.n, self.g, self.trigger, cg, cs):
            # partials FIFO, skipping groups that cannot open (scheduler.py:322-343)
            for s in list(self.buffer.parts):
                grp = self.carry.get(s.instance_id)
                if grp is None:
                    raise OracleContract("partial without group")
                if s.instance_id not in opened:
                    if len(opened) >= self.n_prime:
                        continue
                    opened[s.instance_id] = grp
                self.buffer.parts.remove(s)
                carried += s.total_tokens
                eng.submit(s)
                log.append(("resumed", s.sample_id))
            keep = []
            for s in self.pending_pool:  # scheduler.py:344-356
                grp = self.carry.get(s.instance_id)
                if s.instance_id in opened or (grp is not None and len(opened) < self.n_prime):
                    opened.setdefault(s.instance_id, grp)
                    eng.submit(s)
                    log.append(("pooled", s.sample_id))
                else:
                    keep.append(s)
            self.pending_pool = keep
            for iid, grp in opened.items():  # scheduler.py:257-263
                if grp.complete:
                    continue
                for o in self.buffer.orph.pop(iid, []):
                    carried += o.total_tokens
                    cs += 1
            while len(opened) < self.n_prime:
                gr = self._new_group()
                opened[gr.instance_id] = gr
                for s in gr.samples:
                    eng.submit(s)
                    log.append(("fresh", s.sample_id))
        while not trigger_fired(self.n, self.g, self.trigger, cg, cs):
            evs = eng.decode_until_event()
            if not evs:
                raise OracleContract("engine drained before the trigger fired")
            for s, _ in evs:
                grp = opened[s.instance_id]
                self._complete(grp)
                cs += 1
                if grp.complete:
                    cg += 1
                    this_step += 1
        done = sorted((gr for gr in opened.values() if gr.complete), key=lambda x: x.completion_seq)
        if len(done) < self.n:
            raise OracleContract("trigger with fewer than N groups")
        batch, surplus = done[: self.n], done[self.n:]
        # park (scheduler.py:372-393)
        back = eng.abort_active()
        paused = [s for s in back if s.status == PAUSED]
        drained = [s for s in back if s.status == PENDING]
        for s in paused:
            if s.paused_at is None or s.segments[-1].version == version:
                s.paused_at = (version, eng.iteration_index, s.instance_id, s.sample_index)
        self.buffer.parts.extend(sorted(paused, key=lambda s: s.paused_at))
        self.buffer.parts.sort(key=lambda s: s.paused_at)
        self.buffer._hw()
        self.pending_pool.extend(sorted(drained, key=lambda s: (s.instance_id, s.sample_index)))
        for gr in surplus:
            self.carry.pop(gr.instance_id, None)
            self.buffer.ready.append(gr)
            self.buffer._hw()
        for gr in opened.values():
            if not gr.complete:
                self.carry[gr.instance_id] = gr
                for s in gr.samples:
                    if s.status == COMPLETED:
                        self.buffer.orph.setdefault(s.instance_id, []).append(s)
                        self.buffer._hw()
        for gr in batch:
            self.carry.pop(gr.instance_id, None)
        return OOutcome(version, batch, eng.clock - c0, eng.cumulative_tokens - t0, carried, this_step,
                        self.buffer.sample_count(), len(self.pending_pool), len(opened), log)

    def undelivered_sample_ids(self):
        return self.buffer.sample_ids() + [s.sample_id for s in self.pending_pool]


# --------------------------------------------------------------------------
# policy functions (policy.py:87-124, 140-198)
# --------------------------------------------------------------------------


def reward_of(sample, target_token):
    """policy.py:103-112."""
    toks = sample.token_ids()
    if sample.finish_reason == STOP_TOKEN:
        toks = toks[:-1]
    if not toks:
        return 0.0
    return sum(1 for t in toks if t == target_token) / len(toks)


def advantages_of(rewards, mode="mean_baseline", eps=1e-6):
    """policy.py:115-124."""
    r = np.asarray(rewards, dtype=float)
    c = r - r.mean()
    if mode == "mean_baseline":
        return c
    return c / (r.std() + eps)


def reinforce_step(logits, samples, adv, lr):
    """Score-function update, policy.py:140-150 + 179-198."""
    z = np.asarray(logits, dtype=float)
    e = np.exp(z - np.max(z))
    p = e / e.sum()
    grad = np.zeros_like(z)
    for s, a in zip(samples, np.asarray(adv, dtype=float)):
        toks = s.token_ids()
        grad += a * (np.bincount(toks, minlength=z.size) - len(toks) * p)
    return z + lr * grad


def make_oracle(cfg: dict):
    """Build an (engine, scheduler) pair from a plain dict config (tests/canon.py schema)."""
    eng = OracleEngine(cfg.get("d0", 0.05), cfg.get("d1", 0.002), cfg["slots"], cfg["l_max"],
                       mode=cfg.get("engine_mode", "length"), seed=cfg.get("seed", 0))
    dist = None
    if cfg.get("engine_mode", "length") == "length":
        d = cfg["dist"]
        dist = TraceDist(d[0], cfg["l_max"], *d[1:])
    sch = OracleScheduler(cfg["n"], cfg["g"], cfg["n_prime"], eng, mode=cfg.get("mode", "april"),
                          trigger=cfg.get("trigger", "groups"), dist=dist, rho=cfg.get("rho", 0.0),
                          seed=cfg.get("seed", 0))
    return eng, sch


# --------------------------------------------------------------------------
# composed k-engine oracle for the data-parallel path
# --------------------------------------------------------------------------


class KEngineOracle:
    """k reference-semantics engines in lockstep behind the single-engine duck type.

    Placement: an instance is placed at its first submit on the rank with the
    fewest active + queued samples (ties to the lowest rank); later submits of
    the same instance are sticky.  Every global iteration each rank admits
    from its own FIFO and advances its own slots; events of one iteration are
    merged rank-major, slot order within a rank.  iteration_index and
    cumulative_tokens are global.  (No reference counterpart exists: the
    reference is a single engine; this composes its semantics.)
    """

    def __init__(self, k, d0, d1, max_slots, l_max, mode="length", seed=0):
        self.engines = [OracleEngine(d0, d1, max_slots, l_max, mode=mode, seed=seed) for _ in range(k)]
        self.k = k
        self.place: dict = {}
        self.iteration_index = 0
        self.cumulative_tokens = 0
        self.clock = 0.0
        self.event_log: list = []

    @property
    def idle(self):
        return all(e.idle for e in self.engines)

    def begin_step(self, version, params=None):
        for e in self.engines:
            e.begin_step(version, params)

    def submit(self, s):
        r = self.place.get(s.instance_id)
        if r is None:
            loads = [len(e.slots) + len(e._queue) for e in self.engines]
            r = loads.index(min(loads))
            self.place[s.instance_id] = r
        self.engines[r].submit(s)

    def decode_until_event(self):
        while True:
            for e in self.engines:
                e._admit()
            live = [e for e in self.engines if e.slots]
            if not live:
                return []
            b = sum(len(e.slots) for e in live)
            self.iteration_index += 1
            self.cumulative_tokens += b
            events = []
            for e in self.engines:  # rank-major
                if e.slots:
                    for s, why in e._advance(1):
                        events.append((s, why))
                        self.event_log.append([self.iteration_index, s.instance_id, s.sample_index, s.total_tokens, why])
            if events:
                return events

    def abort_active(self):
        out = []
        for e in self.engines:
            out.extend(e.abort_active())
        return out


def make_k_oracle(cfg: dict, k: int):
    eng = KEngineOracle(k, cfg.get("d0", 0.05), cfg.get("d1", 0.002), cfg["slots"], cfg["l_max"])
    d = cfg["dist"]
    sch = OracleScheduler(cfg["n"], cfg["g"], cfg["n_prime"], eng, mode=cfg.get("mode", "april"),
                          trigger=cfg.get("trigger", "groups"), dist=TraceDist(d[0], cfg["l_max"], *d[1:]),
                          rho=cfg.get("rho", 0.0), seed=cfg.get("seed", 0))
    return eng, sch
