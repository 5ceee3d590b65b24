"""The B200 decode engine behind the reference's duck-typed `Engine` contract.

Reference contract (src/april_sim/engine.py:98-289; the eight members the
Scheduler touches are listed in SURVEY.md §8b):
  idle, begin_step(version, params), submit(sample), decode_until_event(),
  abort_active(), clock, iteration_index, cumulative_tokens
plus decode_iteration, active_count, queued_count, active_samples, _queue.

Everything per-iteration runs on the GPU (csrc/engine.cu): admission,
token growth / sampling, stop detection, stable compaction, the event log,
group done-counters and the trigger.  This class only mirrors the outcome
onto the caller's RolloutSample objects, exactly as the reference engine
mutates them (status, open_segment, token counts, mark_completed), and
copies a segment's token ids / behaviour log-probs to the host when the
segment closes.

`run_until_trigger` is the fused path the B200 Scheduler uses: one C-ABI
call per RL step decodes until N whole groups are complete with no host
round-trip per token.
"""

from __future__ import annotations

import ctypes as C
import os
from collections import deque
from dataclasses import dataclass

import numpy as np

from . import _capi as capi
from .errors import ConfigError, ContractViolation
from .model import ModelSpec, SamplingConfig, synthetic_prompt
from .rng import LANE_POLICY_TOKENS, key_words, philox_key
from .rollouts import ACTIVE, COMPLETED, PAUSED, PENDING, RolloutSample


@dataclass(frozen=True)
class EngineConfig:
    """Same fields and validation as engine.py:38-66.

    On the GPU `d0`/`d1` no longer drive the clock (time is measured); they
    remain the cost model the idle-fraction metric is quoted against.
    """

    d0: float = 0.05
    d1: float = 0.002
    max_slots: int = 64
    l_max: int = 16384

    def __post_init__(self) -> None:
        if self.d0 < 0:
            raise ConfigError(f"d0 must be >= 0, got {self.d0}")
        if self.d1 <= 0:
            raise ConfigError(f"d1 must be > 0, got {self.d1}")
        if self.max_slots < 1:
            raise ConfigError(f"max_slots must be >= 1, got {self.max_slots}")
        if self.l_max < 1:
            raise ConfigError(f"l_max must be >= 1, got {self.l_max}")

    def aggregate_rate(self, batch: int) -> float:
        return 0.0 if batch <= 0 else batch / (self.d0 + self.d1 * batch)

    @property
    def peak_rate(self) -> float:
        return self.aggregate_rate(self.max_slots)


@dataclass(frozen=True)
class Event:
    clock: float
    sample: RolloutSample
    tokens: int
    reason: str
    iteration: int = -1

    @property
    def sample_id(self) -> str:
        return self.sample.sample_id

    def to_record(self) -> dict:
        return {"clock": self.clock, "sample_id": self.sample_id, "tokens": self.tokens, "reason": self.reason,
                "iteration_index": self.iteration}


_TRIGGER_MODES = {"groups": 0, "samples": 1}


class Engine:
    """GPU engine.  Subclasses pick the stop rule and the model."""

    _stop_mode = capi.STOP_TRACE
    _model_kind = capi.MODEL_NONE

    def __init__(self, config: EngineConfig, *, global_seed: int = 0, model: ModelSpec | None = None,
                 sampling: SamplingConfig | None = None, max_handles: int | None = None,
                 max_groups: int | None = None, device: int = 0, record_payload: bool | None = None,
                 prompt_len: int = 256, page_size: int = 16, kv_pages: int = 0, weight_seed: int = 0,
                 weight_std: float = 0.02, prompt_source=None, nondeterministic_gemm: bool = False,
                 kv_resume: str = "retain", gemm_autotune: bool = True):
        self.config = config
        self.global_seed = global_seed
        self.model = model
        self.sampling = sampling or SamplingConfig()
        if model is not None:
            self._model_kind = capi.MODEL_TRANSFORMER
        self.device = device
        self.max_handles = max_handles or max(4096, 8 * config.max_slots)
        self.max_groups = max_groups or self.max_handles
        self.prompt_len = prompt_len
        self.page_size = page_size
        self.kv_pages = kv_pages
        self.weight_seed, self.weight_std = weight_seed, weight_std
        # fp32 residual GEMMs may split K with TMA reduce-add (faster at mid-size batches; the split
        # summation order is then not fixed run to run)
        self.nondeterministic_gemm = bool(nondeterministic_gemm)
        # "retain": a paused partial keeps its KV pages across steps (exact while weights are fixed);
        # "reprefill": the abort drops them and the resume re-prefills prompt + carried tokens, the
        # cost APRIL pays when the policy weights change between steps
        if kv_resume not in ("retain", "reprefill"):
            raise ConfigError(f"kv_resume must be 'retain' or 'reprefill', not {kv_resume!r}")
        self.kv_resume = kv_resume
        # time the decode GEMM schedules on this GPU at creation (cached per process and shape)
        self.gemm_autotune = bool(gemm_autotune)
        self.prompt_source = prompt_source or (
            lambda iid: synthetic_prompt(global_seed, iid, prompt_len, model.vocab)) if model else None
        if record_payload is None:
            record_payload = self._model_kind != capi.MODEL_NONE
        self._record = bool(record_payload) and self._model_kind != capi.MODEL_NONE
        self._h = None  # device engine (created lazily for the context-free model)
        self._n_symbols = 0
        self.version = 0
        self.iteration_index = 0
        self.cumulative_tokens = 0
        self._queue: deque = deque()
        self._active: dict[int, RolloutSample] = {}
        self._handle: dict[int, int] = {}      # id(sample) -> handle
        self._by_handle: dict[int, RolloutSample] = {}
        self._free = list(range(self.max_handles - 1, -1, -1))
        self._gslot: dict[int, int] = {}       # instance_id -> group slot
        self._grefs: dict[int, int] = {}
        self._gfree = list(range(self.max_groups - 1, -1, -1))
        self._pending: list = []
        self.last_run = None
        self._h2d = self._d2h = 0  # bytes crossing PCIe through this API (bench e2e accounting)
        self.last_admitted: list = []  # admissions of the last device call, in FIFO order
        self.last_admit_iterations: list = []  # their iteration_index (before the admitting iteration)
        self.dp_world = 1
        if self._model_kind != capi.MODEL_CONTEXT_FREE:
            self._create()

    # -- device engine ---------------------------------------------------------------

    def _create(self, n_symbols: int = 0) -> None:
        c = capi.EngineConfigC()
        c.max_slots, c.l_max = self.config.max_slots, self.config.l_max
        c.max_handles, c.max_groups = self.max_handles, self.max_groups
        c.stop_mode, c.model_kind, c.n_symbols = self._stop_mode, self._model_kind, n_symbols
        c.page_size, c.kv_pages, c.max_prompt = self.page_size, self.kv_pages, self.prompt_len
        s = self.sampling
        c.temperature, c.top_p, c.greedy = s.temperature, s.top_p, int(s.greedy)
        c.n_eos = len(s.eos_ids)
        for i, t in enumerate(s.eos_ids):
            c.eos_ids[i] = t
        c.record_payload = int(self._record)
        c.weight_seed, c.weight_std = self.weight_seed, self.weight_std
        c.nondeterministic_gemm = int(self.nondeterministic_gemm)
        c.kv_resume = int(self.kv_resume == "reprefill")
        c.gemm_autotune = int(self.gemm_autotune)
        m = None
        if self.model is not None:
            sp = self.model
            m = capi.ModelConfig(sp.n_layers, sp.d_model, sp.n_q_heads, sp.n_kv_heads, sp.head_dim, sp.d_ff,
                                 sp.vocab, int(sp.qkv_bias), int(sp.qk_norm), int(sp.tied_embeddings),
                                 sp.rope_theta, sp.norm_eps)
        h = C.c_void_p()
        capi.call("ab_engine_create", C.byref(c), C.byref(m) if m is not None else None, self.device, C.byref(h))
        self._h = h
        self._n_symbols = n_symbols
        n_cap = self.max_handles + self.config.max_slots
        self._ev_buf = (capi.Event * n_cap)()
        self._adm_buf = (capi.Admit * n_cap)()

    def close(self) -> None:
        if self._h is not None:
            capi.lib().ab_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- bookkeeping ------------------------------------------------------------------

    @property
    def active_count(self) -> int:
        return len(self._active)

    @property
    def queued_count(self) -> int:
        return len(self._queue)

    @property
    def idle(self) -> bool:
        return not self._active and not self._queue

    def active_samples(self) -> list[RolloutSample]:
        return list(self._active.values())

    @property
    def clock(self) -> float:
        """Device wall-clock seconds since the engine was created (globaltimer)."""
        if self._h is None:
            return 0.0
        st = capi.Stats()
        capi.call("ab_engine_stats", self._h, C.byref(st))
        return st.clock

    def stats(self) -> capi.Stats:
        st = capi.Stats()
        capi.call("ab_engine_stats", self._h, C.byref(st))
        return st

    def begin_step(self, version: int, params=None) -> None:
        if not self.idle:
            raise ContractViolation("begin_step requires an idle engine")
        logits_ptr = None
        if self._model_kind == capi.MODEL_CONTEXT_FREE:
            if params is None:
                raise ContractViolation("policy-driven decode needs policy parameters")
            z = np.ascontiguousarray(getattr(params, "logits", params), dtype=np.float64)
            if z.ndim != 1 or z.size < 2:
                raise ConfigError("logits must be a vector over >= 1 token plus STOP")
            if self._h is None:
                self._create(z.size)
            elif z.size != self._n_symbols:
                raise ConfigError(f"vocabulary changed from {self._n_symbols - 1} to {z.size - 1}")
            self._logits = z
            logits_ptr = z.ctypes.data_as(capi.F64P)
        capi.call("ab_engine_begin_step", self._h, int(version), logits_ptr)
        self.version = version

    # -- admission ---------------------------------------------------------------------

    def _acquire(self, sample: RolloutSample) -> int:
        h = self._handle.get(id(sample))
        if h is not None:
            return h
        if not self._free:
            raise ContractViolation("no free sample handles (raise max_handles)")
        h = self._free.pop()
        self._handle[id(sample)] = h
        self._by_handle[h] = sample
        iid = sample.instance_id
        if iid not in self._gslot:
            if not self._gfree:
                raise ContractViolation("no free group slots (raise max_groups)")
            g = self._gfree.pop()
            self._gslot[iid] = g
            self._grefs[iid] = 0
            if self._model_kind == capi.MODEL_TRANSFORMER:
                self._flush()
                prompt = np.ascontiguousarray(self.prompt_source(iid), dtype=np.int32)
                capi.call("ab_engine_open_group", self._h, g, prompt.ctypes.data_as(capi.I32P), int(prompt.size))
                self._h2d += prompt.nbytes
        self._grefs[iid] += 1
        return h

    def _release(self, samples) -> None:
        hs = []
        for s in samples:
            h = self._handle.pop(id(s), None)
            if h is None:
                continue
            del self._by_handle[h]
            hs.append(h)
            iid = s.instance_id
            self._grefs[iid] -= 1
            if self._grefs[iid] == 0:
                g = self._gslot.pop(iid)
                del self._grefs[iid]
                if self._model_kind == capi.MODEL_TRANSFORMER:
                    self._flush()
                    capi.call("ab_engine_release_group", self._h, g)
                self._gfree.append(g)
        if hs:
            arr = (C.c_int32 * len(hs))(*hs)
            capi.call("ab_engine_release", self._h, arr, len(hs))
            self._free.extend(reversed(hs))

    def submit(self, sample: RolloutSample) -> None:
        if sample.status not in (PENDING, PAUSED):
            raise ContractViolation(f"cannot submit sample {sample.sample_id} with status {sample.status!r}")
        h = self._acquire(sample)
        if self._stop_mode == capi.STOP_TRACE:
            stop_at = -1 if sample.target_length is None else min(int(sample.target_length), self.config.l_max)
        else:
            stop_at = -1
        k0, k1 = key_words(philox_key(self.global_seed, LANE_POLICY_TOKENS, sample.instance_id,
                                      sample.sample_index))
        self._pending.append((h, self._gslot[sample.instance_id], sample.total_tokens, stop_at, k0, k1))
        self._queue.append(sample)

    def _flush(self) -> None:
        if not self._pending:
            return
        n = len(self._pending)
        arr = (capi.SampleDesc * n)(*[capi.SampleDesc(*p) for p in self._pending])
        self._pending = []
        capi.call("ab_engine_submit", self._h, arr, n)
        self._h2d += C.sizeof(arr)

    # -- decode ------------------------------------------------------------------------

    def decode_iteration(self) -> list[Event]:
        return self._run(capi.RunArgs(max_iters=1))

    def decode_until_event(self) -> list[Event]:
        return self._run(capi.RunArgs(stop_on_event=1))

    def set_iteration(self, iteration_index: int) -> None:
        """Align the device iteration counter with a global (data-parallel) index."""
        capi.call("ab_engine_set_iteration", self._h, int(iteration_index))
        self.iteration_index = int(iteration_index)

    def set_counters(self, iteration_index: int, cumulative_tokens: int) -> None:
        capi.call("ab_engine_set_counters", self._h, int(iteration_index), int(cumulative_tokens))
        self.iteration_index, self.cumulative_tokens = int(iteration_index), int(cumulative_tokens)

    def dp_attach(self, comm, timeout_ms: int = 60_000) -> None:
        """Join the device-side lockstep exchange of `comm.world` engines (one per GPU).

        Every rank exports its exchange buffer; the (pid, device pointer, CUDA IPC handle) triples
        are all-gathered once; a peer in this process is attached by pointer, a peer in another
        process through its IPC handle (NVLink P2P on one node).  After this every decode
        iteration ends with the peer-memory exchange kernel, so `run_until_trigger` /
        `run_until_drained` / `decode_until_event` decide trigger and drain globally on the device.
        """
        if comm.world < 2:
            return
        if self._h is None:
            raise ContractViolation("dp_attach needs the device engine (the context-free model creates it at its "
                                    "first begin_step)")
        ptr = C.c_uint64()
        ipc = (C.c_uint8 * 64)()
        capi.call("ab_engine_dp_export", self._h, comm.world, C.byref(ptr), ipc)
        mine = (os.getpid(), int(ptr.value), bytes(ipc))
        peers_info = comm.allgather(mine)
        peers = (capi.DpPeer * comm.world)()
        for r, (pid, p, h) in enumerate(peers_info):
            peers[r].ptr = p
            peers[r].kind = 0 if pid == os.getpid() else 1
            C.memmove(peers[r].ipc, h, 64)
        capi.call("ab_engine_dp_attach", self._h, comm.world, comm.rank, peers, int(timeout_ms))
        comm.allgather(None)  # every rank attached before any exchange
        self.dp_world = comm.world

    def dp_detach(self) -> None:
        if self.dp_world > 1:
            capi.call("ab_engine_dp_detach", self._h)
            self.dp_world = 1

    def decode_iterations(self, k: int) -> list[Event]:
        """Run up to k decode iterations in one device call (stops early only if drained)."""
        return self._run(capi.RunArgs(max_iters=int(k)))

    def run_until_trigger(self, n: int, g: int, trigger: str, completed_groups: int, completed_samples: int,
                          group_done: dict[int, int] | None = None) -> list[Event]:
        """Fused APRIL loop: decode until check_trigger(n, g, trigger) fires (scheduler.py:272-283)."""
        self._preset_groups(group_done or {})
        return self._run(capi.RunArgs(use_trigger=1, trigger_mode=_TRIGGER_MODES[trigger], n_target=n,
                                      group_size=g, completed_groups=completed_groups,
                                      completed_samples=completed_samples), refresh=False)

    def run_until_drained(self, g: int, group_done: dict[int, int] | None = None) -> list[Event]:
        """Synchronous baseline loop: decode until every submitted sample finished (scheduler.py:208-214)."""
        self._preset_groups(group_done or {})
        return self._run(capi.RunArgs(group_size=g), refresh=False)

    def _preset_groups(self, group_done: dict[int, int]) -> None:
        pairs = [(self._gslot[iid], cnt) for iid, cnt in group_done.items() if iid in self._gslot]
        if pairs:
            flat = (C.c_int32 * (2 * len(pairs)))(*[x for p in pairs for x in p])
            capi.call("ab_engine_set_group_done", self._h, flat, len(pairs))

    def _run(self, args: capi.RunArgs, refresh: bool = True) -> list[Event]:
        if self._h is None:
            return []
        self._flush()
        res = capi.RunResult()
        cap = len(self._ev_buf)
        capi.call("ab_engine_run", self._h, C.byref(args), C.byref(res), self._ev_buf, cap, self._adm_buf, cap)
        self._d2h += C.sizeof(res) + res.n_events * C.sizeof(capi.Event) + res.n_admits * C.sizeof(capi.Admit)
        self.last_run = res
        self.iteration_index = res.iteration_index
        self.cumulative_tokens = res.cumulative_tokens
        events = self._apply_logs(res)
        if refresh and self._active:
            self._refresh_active()
        return events

    def _apply_logs(self, res) -> list[Event]:
        adm, evs = self._adm_buf, self._ev_buf
        na, ne = res.n_admits, res.n_events
        i = j = 0
        out: list[Event] = []
        finished: list[RolloutSample] = []
        self.last_admitted = []
        self.last_admit_iterations = []
        with_tokens = self._record
        while i < na or j < ne:
            # admissions of iteration k (logged with index k) precede finishes of iteration k (index k+1)
            if i < na and (j >= ne or adm[i].iteration < evs[j].iteration):
                s = self._by_handle[adm[i].handle]
                q = self._queue.popleft()
                if q is not s:
                    raise ContractViolation("host queue mirror out of sync with the device FIFO")
                s.status = ACTIVE
                s.open_segment(self.version, with_tokens=with_tokens)
                self._active[id(s)] = s
                self.last_admitted.append(s)
                self.last_admit_iterations.append(adm[i].iteration)
                i += 1
            else:
                e = evs[j]
                s = self._by_handle[e.handle]
                seg = s.segments[-1]
                seg.token_count = e.tokens - (s.total_tokens - seg.token_count)
                reason = capi.REASONS[e.reason]
                s.mark_completed(self.version, reason)
                del self._active[id(s)]
                finished.append(s)
                out.append(Event(e.clock, s, e.tokens, reason, e.iteration))
                j += 1
        if finished:
            if with_tokens:
                self._materialize(finished)
            self._release(finished)
        return out

    def _refresh_active(self) -> None:
        b = len(self._active)
        hs = (C.c_int32 * b)()
        gen = (C.c_int32 * b)()
        n = C.c_int()
        capi.call("ab_engine_active", self._h, hs, gen, b, C.byref(n))
        for k in range(n.value):
            s = self._by_handle[hs[k]]
            seg = s.segments[-1]
            seg.token_count = gen[k] - (s.total_tokens - seg.token_count)

    def _materialize(self, samples) -> None:
        """Copy each sample's open segment payload (device -> host lists)."""
        n = len(samples)
        hs = (C.c_int32 * n)()
        st = (C.c_int32 * n)()
        ct = (C.c_int32 * n)()
        for k, s in enumerate(samples):
            seg = s.segments[-1]
            hs[k] = self._handle[id(s)]
            st[k] = s.total_tokens - seg.token_count
            ct[k] = seg.token_count
        total = sum(ct)
        self._d2h += total * 12
        tok = np.empty(max(total, 1), dtype=np.int32)
        lp = np.empty(max(total, 1), dtype=np.float64)
        capi.call("ab_engine_read_payload", self._h, hs, st, ct, n, tok.ctypes.data_as(capi.I32P),
                  lp.ctypes.data_as(capi.F64P))
        o = 0
        for k, s in enumerate(samples):
            seg = s.segments[-1]
            c = ct[k]
            seg.tokens = tok[o:o + c].tolist()
            seg.behavior_logprobs = lp[o:o + c].tolist()
            o += c

    # -- abort ----------------------------------------------------------------------------

    def abort_active(self) -> list[RolloutSample]:
        if self._h is None:
            return []
        self._flush()
        cap = len(self._active) + len(self._queue)
        hs = (C.c_int32 * max(cap, 1))()
        gen = (C.c_int32 * max(cap, 1))()
        na, nq = C.c_int(), C.c_int()
        capi.call("ab_engine_abort", self._h, hs, gen, max(cap, 1), C.byref(na), C.byref(nq))
        self._d2h += 8 * (na.value + nq.value)
        out: list[RolloutSample] = []
        paused = []
        for k in range(na.value):
            s = self._by_handle[hs[k]]
            seg = s.segments[-1]
            seg.token_count = gen[k] - (s.total_tokens - seg.token_count)
            s.status = PAUSED
            out.append(s)
            paused.append(s)
        drained = []
        for k in range(na.value, na.value + nq.value):
            s = self._by_handle[hs[k]]
            out.append(s)
            if not s.segments:
                drained.append(s)
        if paused and self._record:
            self._materialize(paused)
        self._active.clear()
        self._queue.clear()
        self._release(drained)  # zero-token samples hold no device state worth keeping
        return out

    def score(self, prompts, responses) -> list:
        """Teacher-forced log-probs (at the engine's temperature) of each response token under the
        CURRENT weights: the trainer's recompute of pi_theta on a mixed-policy batch (
        policy.py:157-176 uses it against the behaviour log-probs).  prompts / responses: sequences of
        token ids; returns one float64 array per response."""
        if self._model_kind != capi.MODEL_TRANSFORMER:
            raise ContractViolation("scoring needs the transformer model")
        if len(prompts) != len(responses):
            raise ContractViolation("score: one prompt per response")
        n = len(prompts)
        if n == 0:
            return []
        self._flush()
        seqs = [np.concatenate([np.asarray(p, dtype=np.int32), np.asarray(r, dtype=np.int32)])
                for p, r in zip(prompts, responses)]
        toks = np.ascontiguousarray(np.concatenate(seqs), dtype=np.int32)
        offs = np.zeros(n + 1, dtype=np.int64)
        offs[1:] = np.cumsum([len(s) for s in seqs])
        plen = np.ascontiguousarray([len(p) for p in prompts], dtype=np.int32)
        nres = [len(r) for r in responses]
        out = np.empty(sum(nres), dtype=np.float64)
        capi.call("ab_engine_score", self._h, toks.ctypes.data_as(capi.I32P),
                  offs.ctypes.data_as(C.POINTER(C.c_int64)), plen.ctypes.data_as(capi.I32P), n,
                  out.ctypes.data_as(capi.F64P))
        self._h2d += toks.nbytes + offs.nbytes + plen.nbytes
        self._d2h += out.nbytes
        return list(np.split(out, np.cumsum(nres)[:-1]))

    def recompute_logprobs(self, samples) -> list:
        """score() of delivered samples against their prompts (prompt_source) and generated tokens."""
        return self.score([self.prompt_source(s.instance_id) for s in samples], [s.token_ids() for s in samples])

    def sequence_logprobs(self, samples):
        """(sum of behaviour log-probs over all generated tokens, token count) per sample, reduced
        on the device from the resident partial-rollout payload (GSPO's length-normalised sequence
        log-ratio uses sum / count).  Samples must still hold their device handle (active, queued
        or paused in the continuation buffer)."""
        n = len(samples)
        if n == 0 or self._h is None:
            return np.zeros(0), np.zeros(0, dtype=np.int32)
        self._flush()
        hs = np.empty(n, dtype=np.int32)
        for k, s in enumerate(samples):
            h = self._handle.get(id(s))
            if h is None:
                raise ContractViolation("sample has no device payload (already delivered or never admitted)")
            hs[k] = h
        sums = np.empty(n, dtype=np.float64)
        lens = np.empty(n, dtype=np.int32)
        capi.call("ab_engine_sequence_logprobs", self._h, hs.ctypes.data_as(capi.I32P), n,
                  sums.ctypes.data_as(capi.F64P), lens.ctypes.data_as(capi.I32P))
        self._d2h += n * 12
        return sums, lens

    def io_bytes(self) -> tuple[int, int]:
        """(host->device, device->host) bytes moved through the C-ABI so far."""
        return self._h2d, self._d2h

    def discard(self, samples) -> None:
        """Release device state (handles, KV pages) of samples leaving the engine for good."""
        self._release(samples)

    # -- weights ------------------------------------------------------------------------------

    def export_weights(self) -> dict:
        """Device bf16 parameters as CPU torch.bfloat16 tensors (for the oracle / checkpoints)."""
        import torch

        n = C.c_int()
        capi.call("ab_engine_weight_count", self._h, C.byref(n))
        out = {}
        name = C.create_string_buffer(128)
        for i in range(n.value):
            r, c = C.c_int64(), C.c_int64()
            capi.call("ab_engine_weight_info", self._h, i, name, 128, C.byref(r), C.byref(c))
            buf = np.empty(r.value * c.value, dtype=np.uint16)
            capi.call("ab_engine_get_weight", self._h, i, buf.ctypes.data_as(C.c_void_p), buf.nbytes)
            out[name.value.decode()] = torch.from_numpy(buf.view(np.int16)).view(torch.bfloat16).view(r.value,
                                                                                                    c.value)
        return out

    def load_weights(self, tensors: dict) -> None:
        """Install new policy weights (the weight-version swap between RL steps).
        `tensors` maps export_weights() names to bf16 tensors of exactly the exported shape (host or
        device).  Layout: "layers.{l}.wqkv" stacks the q, k, v projection rows; "layers.{l}.wgu" is
        tile-interleaved -- per 128-row tile, 64 gate rows then the matching 64 up rows (an HF-style
        [gate; up] concatenation must be re-tiled first, see oracle/cpu_model.py:split_gate_up for
        the inverse).  Call between steps.  Only with kv_resume="reprefill": the next
        begin_step(version) recomputes the resident prompt KV and resumed partials are re-prefilled
        under the new weights.  With kv_resume="retain" resident KV would silently mix old-policy
        keys/values with the new weights, so a swap while any prompt group (or parked partial) is
        resident is refused."""
        import torch

        if not self.idle:
            raise ContractViolation("load_weights requires an idle engine")
        if self.kv_resume == "retain" and (self._gslot or self._handle):
            raise ContractViolation("load_weights with kv_resume='retain' while KV is resident (prompt groups or "
                                    "parked partials computed under the old weights); use kv_resume='reprefill' "
                                    "or discard them first")
        n = C.c_int()
        capi.call("ab_engine_weight_count", self._h, C.byref(n))
        name = C.create_string_buffer(128)
        index = {}
        for i in range(n.value):
            r, c = C.c_int64(), C.c_int64()
            capi.call("ab_engine_weight_info", self._h, i, name, 128, C.byref(r), C.byref(c))
            index[name.value.decode()] = (i, r.value, c.value)
        for k, t in tensors.items():
            if k not in index:
                raise ConfigError(f"unknown weight {k!r}")
            i, r, c = index[k]
            t = t.detach().to(torch.bfloat16).contiguous()
            if tuple(t.shape) != (r, c):
                raise ConfigError(f"weight {k!r}: expected {r}x{c}, got {tuple(t.shape)}")
            capi.call("ab_engine_set_weight", self._h, i, C.c_void_p(t.data_ptr()), r * c * 2)
            if not t.is_cuda:
                self._h2d += r * c * 2

    def release_memory(self) -> None:
        """Free the KV pool of an idle engine (kv_resume="reprefill") so a co-located trainer can use
        the HBM between rollout steps (torch_memory_saver-style pause)."""
        capi.call("ab_engine_release_memory", self._h)

    def resume_memory(self) -> None:
        """Re-acquire the KV pool; resident prompt KV is recomputed by the next submit."""
        capi.call("ab_engine_resume_memory", self._h)

    # -- profiling ---------------------------------------------------------------------------

    def profile(self, enable: bool = True, sample_every: int = 8) -> None:
        capi.call("ab_engine_profile", self._h, int(enable), int(sample_every))

    def kernel_stats(self) -> list[dict]:
        buf = (capi.KernelStat * 64)()
        n = C.c_int()
        capi.call("ab_engine_kernel_stats", self._h, buf, 64, C.byref(n))
        return [{"name": buf[i].name.decode(), "launches": buf[i].launches, "ms": buf[i].ms,
                 "bytes": buf[i].bytes, "flops": buf[i].flops} for i in range(min(n.value, 64))]


class LengthDrivenEngine(Engine):
    """Sequences stop at a pre-drawn target length or l_max (engine.py:214-240).

    With `model=None` the GPU only advances counters (exact replay of the
    reference's length-driven engine); with a ModelSpec every iteration is a
    real transformer decode step whose tokens are sampled but whose stop is
    dictated by the trace (the bit-exact replay mode of the north star).
    """

    _stop_mode = capi.STOP_TRACE


class PolicyDrivenEngine(Engine):
    """Sequences stop when the policy draws STOP/EOS or at l_max (engine.py:243-289).

    Without a ModelSpec the policy is the reference's context-free softmax
    over V tokens + STOP, evaluated and sampled on the GPU.
    """

    _stop_mode = capi.STOP_POLICY

    def __init__(self, config: EngineConfig, global_seed: int = 0, **kw):
        if kw.get("model") is None:
            self._model_kind = capi.MODEL_CONTEXT_FREE
        super().__init__(config, global_seed=global_seed, **kw)
