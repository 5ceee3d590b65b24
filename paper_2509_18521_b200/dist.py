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

Two lockstep implementations share the placement, mirrors and log merge:

* device lockstep (`GpuLocal` after `Engine.dp_attach`, the GPU path): the
  per-iteration sum runs on the device.  Every captured decode iteration
  ends with `k_dp_exchange` (csrc/engine.cu), which stores this rank's
  counts into every peer's exchange buffer over NVLink (CUDA IPC) and sums
  the world's records, so each rank's device loop knows the global trigger,
  drain, iteration_index and cumulative_tokens — one `ab_engine_run` per
  scheduler call, no host round trip per iteration.
* host lockstep (`OracleLocal`, the CPU tests): one host allreduce per
  iteration through `Comm`.

The host collectives are abstract (`Comm`): `TorchComm` uses
torch.distributed (NCCL on GPUs, gloo in the CPU tests), `ThreadComm` joins
several engines of one process (one thread each; the one-GPU tests).
`gather_responses` gathers the finished responses (int32 token ids, fp64
behaviour log-probs, lengths) to the trainer over the same collectives.
Parity: the composed k-engine oracle (oracle/sim_ref.py KEngineOracle) —
tests/test_dp.py (gloo, CPU) and tests/test_dp_gpu.py (device lockstep)
compare canonical step records bit for bit.
"""

from __future__ import annotations

import threading
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


class ThreadComm(Comm):
    """In-process collectives between `world` threads (one engine per thread)."""

    class _Shared:
        def __init__(self, world, timeout):
            self.world = world
            self.barrier = threading.Barrier(world, timeout=timeout)
            self.slots = [None] * world

    def __init__(self, shared: "ThreadComm._Shared", rank: int):
        self.shared, self.rank, self.world = shared, rank, shared.world

    @classmethod
    def group(cls, world, timeout: float = 300.0):
        sh = cls._Shared(world, timeout)
        return [cls(sh, r) for r in range(world)]

    def abort(self):
        """Break the group's barrier (a failing thread releases the others)."""
        self.shared.barrier.abort()

    def allgather(self, obj):
        sh = self.shared
        sh.barrier.wait()
        sh.slots[self.rank] = obj
        sh.barrier.wait()
        out = list(sh.slots)
        sh.barrier.wait()
        return out

    def allreduce_sum(self, vals):
        return [sum(x) for x in zip(*self.allgather(list(vals)))]


def gather_responses(comm: Comm, samples):
    """Finished-response gather to the trainer (once per step).

    `samples` is the delivered batch (same order on every rank).  A rank owns
    the samples it generated (every segment carries its payload; a remote
    mirror's segments carry none).  Returns, in delivered order, (token ids,
    behaviour log-probs) per sample.  Over `TorchComm` the payload moves as
    three flat tensors per rank (int64 [index, length] pairs, int32 token
    ids, fp64 log-probs) with torch.distributed all_gather — NCCL over
    NVLink on GPUs (CUDA tensors), gloo on CPU.
    """
    own_idx, own_tok, own_lp = [], [], []
    for k, s in enumerate(samples):
        if s.segments and all(seg.tokens is not None for seg in s.segments):
            own_idx.append(k)
            own_tok.append(s.token_ids())
            own_lp.append(s.behavior_logprob_trace())
    out = [None] * len(samples)
    if comm.world == 1 or not isinstance(comm, TorchComm):
        parts = comm.allgather((own_idx, own_tok, own_lp))
        for idx, tok, lp in parts:
            for k, t, l in zip(idx, tok, lp):
                out[k] = (t, l)
    else:
        torch, dist = comm.torch, comm.dist
        dev = comm.device
        n_own, t_own = len(own_idx), sum(len(t) for t in own_tok)
        sizes = torch.tensor([n_own, t_own], dtype=torch.int64, device=dev)
        all_sizes = [torch.zeros_like(sizes) for _ in range(comm.world)]
        dist.all_gather(all_sizes, sizes, group=comm.group)
        all_sizes = [tuple(int(x) for x in t.tolist()) for t in all_sizes]
        max_n = max(1, max(n for n, _ in all_sizes))
        max_t = max(1, max(t for _, t in all_sizes))
        meta = torch.zeros(max_n, 2, dtype=torch.int64)
        tok = torch.zeros(max_t, dtype=torch.int32)
        lp = torch.zeros(max_t, dtype=torch.float64)
        o = 0
        for j, (k, t, l) in enumerate(zip(own_idx, own_tok, own_lp)):
            meta[j, 0], meta[j, 1] = k, len(t)
            tok[o:o + len(t)] = torch.tensor(t, dtype=torch.int32)
            lp[o:o + len(t)] = torch.tensor(l, dtype=torch.float64)
            o += len(t)
        pin = str(dev).startswith("cuda")
        bufs = []
        for x in (meta, tok, lp):
            x = x.pin_memory().to(dev, non_blocking=True) if pin else x
            parts = [torch.empty_like(x) for _ in range(comm.world)]
            dist.all_gather(parts, x, group=comm.group)
            bufs.append([p.cpu() for p in parts])
        for r, (n_r, _) in enumerate(all_sizes):
            m, tk, l = bufs[0][r], bufs[1][r], bufs[2][r]
            o = 0
            for j in range(n_r):
                k, ln = int(m[j, 0]), int(m[j, 1])
                out[k] = (tk[o:o + ln].tolist(), l[o:o + ln].tolist())
                o += ln
    if any(x is None for x in out):
        raise ContractViolation("finished-response gather: a delivered sample has no owner")
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
        if getattr(self.local, "device_lockstep", False):
            return self._run_device(stop_on_event, trigger, max_iters)
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

    def _run_device(self, stop_on_event, trigger, max_iters):
        """One device call: the lockstep loop with the per-iteration exchange on the GPUs."""
        adm, evs, it, cum = self.local.run_lockstep(self.iteration_index, self.cumulative_tokens,
                                                    stop_on_event, trigger, self._g_size, self._g_done,
                                                    max_iters)
        adm_log = [(i, s.instance_id, s.sample_index) for s, i in adm]
        ev_log = [(ev.iteration, ev.sample.instance_id, ev.sample.sample_index, ev.tokens,
                   _CODE[ev.reason]) for ev in evs]
        self.iteration_index, self.cumulative_tokens = it, cum
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
    """LocalAdapter over this rank's B200 engine.

    After `attach(comm)` (device lockstep) a scheduler call is one `ab_engine_run`: the decode
    iterations end with the peer-memory exchange, so the trigger / drain are global on the device.
    Without it, one device iteration per global iteration with a host allreduce in between.
    """

    def __init__(self, engine):
        self.e = engine
        self._queued_ids = set()

    def attach(self, comm, timeout_ms: int = 60_000):
        self.e.dp_attach(comm, timeout_ms)
        return self

    @property
    def device_lockstep(self):
        return self.e.dp_world > 1

    def run_lockstep(self, iteration_index, cumulative_tokens, stop_on_event, trigger, g, g_done, max_iters):
        from . import _capi as capi
        from .engine import _TRIGGER_MODES

        e = self.e
        e.set_counters(iteration_index, cumulative_tokens)
        e._preset_groups(g_done)
        if trigger is not None:
            n, g, mode, cg, cs = trigger
            args = capi.RunArgs(use_trigger=1, trigger_mode=_TRIGGER_MODES[mode], n_target=n, group_size=g,
                                completed_groups=cg, completed_samples=cs)
        else:
            args = capi.RunArgs(group_size=g, stop_on_event=int(stop_on_event), max_iters=int(max_iters))
        evs = e._run(args, refresh=stop_on_event)
        adm = list(zip(e.last_admitted, e.last_admit_iterations))
        return adm, evs, e.last_run.iteration_index, e.last_run.cumulative_tokens

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


