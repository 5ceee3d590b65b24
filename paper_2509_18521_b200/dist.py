"""Data-parallel APRIL rollout: one engine per GPU, lockstep iterations.

SURVEY.md §8e.  Groups are independent, so the path shards by prompt group:
every rank runs the same (replicated, deterministic) Scheduler and owns the
samples of the groups placed on it.  A new group goes to the rank with the
fewest active + queued samples (ties to the lowest rank); resumed partials
stay where their KV and payload live.  Iterations are global and lockstep:
after each one the ranks sum four integers (groups completed, samples
completed, live batch of this iteration, live batch of the next) — that is
the only per-iteration exchange, and it decides the trigger, the global
iteration_index / cumulative_tokens, and drain.  Once per run the ranks
all-gather their admission and finish logs, so every rank's scheduler sees
the same global event stream (rank-major within an iteration, slot order
within a rank) and applies remote outcomes to its mirror of the remote
samples.

The collective is abstract (`Comm`): `TorchComm` uses torch.distributed
(NCCL on GPUs, gloo in the CPU tests).  The per-iteration sum is issued by
the host here; a device-side version (NCCL inside the captured iteration
graph) is the next step.  Parity: the composed k-engine oracle
(oracle/sim_ref.py KEngineOracle) — tests/test_dp.py runs world_size 2 over
gloo and compares canonical step records bit for bit.
"""

from __future__ import annotations

from collections import deque

from .errors import ContractViolation
from .rollouts import ACTIVE, PAUSED, PENDING

_REASONS = ("stop_token", "target_length", "max_length")
_CODE = {r: i for i, r in enumerate(_REASONS)}


class Comm:
    rank = 0
    world = 1

    def allreduce_sum(self, vals: list[int]) -> list[int]:
        return list(vals)

    def allgather(self, obj) -> list:
        return [obj]


class TorchComm(Comm):
    """torch.distributed collectives (any backend; int64 tensors on `device`)."""

    def __init__(self, group=None, device="cpu"):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group, self.device = torch, dist, group, device
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allreduce_sum(self, vals):
        t = self.torch.tensor(vals, dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return [int(x) for x in t.tolist()]

    def allgather(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


class DataParallelEngine:
    """The reference engine duck type over `comm.world` lockstep engines.

    `local` is this rank's engine adapter (see `LocalAdapter` below): it owns
    only the samples placed on this rank.  All other samples are mirrored
    from the gathered logs.
    """

    def __init__(self, local, comm: Comm, max_slots: int):
        self.local = local
        self.comm = comm
        self.rank, self.world = comm.rank, comm.world
        self.S = max_slots
        self.place: dict[int, int] = {}
        self.load = [0] * self.world  # active + queued samples per rank
        self.version = 0
        self.iteration_index = 0
        self.cumulative_tokens = 0
        self._ids: dict[tuple, object] = {}  # (iid, sidx) -> this rank's sample object
        self._remote_q = [deque() for _ in range(self.world)]
        self._remote_active = [dict() for _ in range(self.world)]
        self._g_done: dict[int, int] = {}
        self._g_size = 0

    # -- duck type ---------------------------------------------------------------------

    @property
    def idle(self):
        return self.local.idle and not any(self._remote_q) and not any(self._remote_active)

    @property
    def clock(self):
        return self.local.clock

    def begin_step(self, version, params=None):
        if not self.idle:
            raise ContractViolation("begin_step requires an idle engine")
        self.version = version
        self.local.begin_step(version, params)

    def submit(self, s):
        if s.status not in (PENDING, PAUSED):
            raise ContractViolation(f"cannot submit sample {s.sample_id} with status {s.status!r}")
        r = self.place.get(s.instance_id)
        if r is None:
            r = self.load.index(min(self.load))
            self.place[s.instance_id] = r
        self.load[r] += 1
        self._ids[(s.instance_id, s.sample_index)] = s
        if r == self.rank:
            self.local.submit(s)
        else:
            self._remote_q[r].append(s)

    def decode_until_event(self):
        return self._run(stop_on_event=True)

    def run_until_trigger(self, n, g, trigger, completed_groups, completed_samples, group_done=None):
        return self._run(trigger=(n, g, trigger, completed_groups, completed_samples), group_done=group_done)

    def run_until_drained(self, g, group_done=None):
        self._g_size = g
        return self._run()

    def abort_active(self):
        local = self.local.abort_active()
        mine = [(s.instance_id, s.sample_index, s.total_tokens, int(s.status == PAUSED and not self._queued(s)))
                for s in local]
        logs = self.comm.allgather(mine)
        out = []
        for r, recs in enumerate(logs):
            for iid, sidx, tokens, active in recs:
                s = self._ids[(iid, sidx)]
                if r != self.rank:
                    if active:
                        seg = s.segments[-1]
                        seg.token_count = tokens - (s.total_tokens - seg.token_count)
                        s.status = PAUSED
                out.append(s)
        for r in range(self.world):
            self._remote_q[r].clear()
            self._remote_active[r].clear()
        self.load = [0] * self.world
        return out

    # -- lockstep loop -----------------------------------------------------------------

    def _queued(self, s):
        return getattr(self.local, "was_queued", lambda _s: False)(s)

    def _run(self, stop_on_event=False, trigger=None, group_done=None, max_iters=0):
        if trigger is not None:
            n, g, mode, cg, cs = trigger
            self._g_size = g
        if group_done is not None:
            self._g_done = {iid: c for iid, c in group_done.items() if self.place.get(iid) == self.rank}
        G = self._g_size
        adm_log, ev_log = [], []
        live_next = self.comm.allreduce_sum([self.local.next_batch()])[0]
        its = 0
        while live_next > 0:
            admitted, events, b = self.local.iterate(self.iteration_index)
            new_g = 0
            for s in admitted:
                adm_log.append((self.iteration_index, s.instance_id, s.sample_index))
            for s, reason in events:
                ev_log.append((self.iteration_index + 1, s.instance_id, s.sample_index, s.total_tokens,
                               _CODE[reason]))
                if G:
                    c = self._g_done.get(s.instance_id, 0) + 1
                    self._g_done[s.instance_id] = c
                    new_g += int(c == G)
            tot = self.comm.allreduce_sum([new_g, len(events), b, self.local.next_batch()])
            self.iteration_index += 1
            self.cumulative_tokens += tot[2]
            live_next = tot[3]
            its += 1
            if trigger is not None:
                cg += tot[0]
                cs += tot[1]
                fired = cg >= n if mode == "groups" else (cs >= n * g and cg >= n)
                if tot[1] > 0 and fired:
                    break
            if stop_on_event and tot[1] > 0:
                break
            if max_iters and its >= max_iters:
                break
        return self._merge(adm_log, ev_log)

    def _merge(self, adm_log, ev_log):
        from .engine import Event

        logs = self.comm.allgather((adm_log, ev_log))
        # remote admissions open segments on the mirrors (in iteration order)
        for r, (adms, _) in enumerate(logs):
            if r == self.rank:
                continue
            for it, iid, sidx in adms:
                s = self._ids[(iid, sidx)]
                q = self._remote_q[r].popleft()
                if q is not s:
                    raise ContractViolation("remote queue mirror out of sync")
                s.status = ACTIVE
                s.open_segment(self.version, with_tokens=False)
                self._remote_active[r][id(s)] = s
        merged = []
        for r, (_, evs) in enumerate(logs):
            for e in evs:
                merged.append((e[0], r, e))
        merged.sort(key=lambda x: (x[0], x[1]))  # stable: slot order within (iteration, rank)
        out = []
        for it, r, (_, iid, sidx, tokens, code) in merged:
            s = self._ids[(iid, sidx)]
            reason = _REASONS[code]
            if r != self.rank:
                seg = s.segments[-1]
                seg.token_count = tokens - (s.total_tokens - seg.token_count)
                s.mark_completed(self.version, reason)
                self._remote_active[r].pop(id(s), None)
            self.load[r] -= 1
            out.append(Event(0.0, s, tokens, reason, it))
        return out


class OracleLocal:
    """LocalAdapter over the CPU oracle engine (used by the gloo tests)."""

    def __init__(self, engine):
        self.e = engine
        self._queued_ids = set()

    @property
    def idle(self):
        return self.e.idle

    @property
    def clock(self):
        return 0.0

    def begin_step(self, version, params=None):
        self.e.begin_step(version, params)

    def submit(self, s):
        self.e.submit(s)

    def next_batch(self):
        return len(self.e.slots) + min(self.e.S - len(self.e.slots), len(self.e._queue))

    def iterate(self, iteration_index):
        before = {id(sl[0]) for sl in self.e.slots}
        self.e._admit()
        admitted = [sl[0] for sl in self.e.slots if id(sl[0]) not in before]
        b = len(self.e.slots)
        events = self.e._advance(1) if b else []
        return admitted, events, b

    def abort_active(self):
        self._queued_ids = {id(s) for s in self.e._queue}
        return self.e.abort_active()

    def was_queued(self, s):
        return id(s) in self._queued_ids


class GpuLocal:
    """LocalAdapter over this rank's B200 engine: one device iteration per global iteration."""

    def __init__(self, engine):
        self.e = engine
        self._queued_ids = set()

    @property
    def idle(self):
        return self.e.idle

    @property
    def clock(self):
        return self.e.clock

    def begin_step(self, version, params=None):
        self.e.begin_step(version, params)

    def submit(self, s):
        self.e.submit(s)

    def next_batch(self):
        a = self.e.active_count
        return a + min(self.e.config.max_slots - a, self.e.queued_count)

    def iterate(self, iteration_index):
        if self.next_batch() == 0:
            return [], [], 0
        self.e.set_iteration(iteration_index)
        evs = self.e.decode_iteration()
        b = self.e.active_count + len(evs)
        return list(self.e.last_admitted), [(ev.sample, ev.reason) for ev in evs], b

    def abort_active(self):
        self._queued_ids = {id(s) for s in self.e._queue}
        return self.e.abort_active()

    def was_queued(self, s):
        return id(s) in self._queued_ids


