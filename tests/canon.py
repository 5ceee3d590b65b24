"""Canonical per-step records shared by the reference golden generator, the
CPU oracle and the B200 engine, so that all three can be compared field by
field (or by digest for the large configurations).

A record captures everything the bit-exact replay contract covers
(SURVEY.md §8a rows a5-a14, Appendix A.3-A.6): the delivered batch and its
completion order, every delivered sample's per-version segments and finish
reason, the outcome counters, the admission log, finish events with their
iteration index, and the state left behind in the continuation buffer and
pending pool.
"""

from __future__ import annotations

import hashlib
import json

REASON = {"stop_token": 0, "target_length": 1, "max_length": 2}
KIND = {"fresh": 0, "resumed": 1, "pooled": 2}

# Replay configurations C1-C5, 1-engine variants.
# dist tuples: (kind, a, b) as in oracle.sim_ref.TraceDist.
CONFIGS = {
    "C1": dict(n=8, g=4, n_prime=16, slots=64, l_max=1024, dist=("lognormal", 5.5, 1.0), rho=0.7, seed=0, steps=20),
    "C2": dict(n=64, g=8, n_prime=128, slots=1024, l_max=4096, dist=("lognormal", 6.6, 1.0), rho=0.7, seed=0, steps=6),
    "C3": dict(n=32, g=8, n_prime=64, slots=64, l_max=16384, dist=("lognormal", 7.5, 1.0), rho=0.7, seed=0, steps=8),
    "C4_1.5": dict(n=32, g=8, n_prime=48, slots=64, l_max=16384, dist=("lognormal", 7.8, 1.2), rho=0.7, seed=0, steps=4),
    "C4_3": dict(n=32, g=8, n_prime=96, slots=64, l_max=16384, dist=("lognormal", 7.8, 1.2), rho=0.7, seed=0, steps=4),
    "C5": dict(n=256, g=16, n_prime=512, slots=1024, l_max=16384, dist=("lognormal", 7.5, 1.0), rho=0.7, seed=0, steps=2),
    # small edge cases: trigger on samples, constant lengths, tiny slot count
    "E_samples": dict(n=3, g=4, n_prime=6, slots=5, l_max=300, dist=("lognormal", 4.0, 1.2), rho=0.3, seed=5,
                      steps=25, trigger="samples"),
    "E_const": dict(n=2, g=2, n_prime=4, slots=16, l_max=1000, dist=("constant", 100, 0), rho=0.0, seed=0, steps=4),
    "E_pool": dict(n=1, g=4, n_prime=3, slots=2, l_max=200, dist=("lognormal", 3.5, 1.0), rho=0.0, seed=3, steps=30),
    "E_cap": dict(n=4, g=3, n_prime=8, slots=24, l_max=120, dist=("lognormal", 4.5, 1.1), rho=0.5, seed=7, steps=40),
}
SYNC_STEPS = {"C1": 5, "C2": 2, "C3": 2, "E_samples": 5, "E_const": 3, "E_cap": 5}

# Toy policy-driven configuration of the reference's own fixtures
# (frontend/tests/fixtures/sample_run/summary.json:12-55).
TOY = dict(n=8, g=8, n_prime=16, slots=128, l_max=64, vocab=4, target=0, lr=0.05, seed=4, steps=60,
           d0=0.05, d1=0.002)


def _seg(s):
    return [[int(seg.version), int(seg.token_count)] for seg in s.segments]


def _sid(sid: str):
    a, b = sid.split(":")
    return [int(a), int(b)]


def sample_record(s, with_tokens=False):
    rec = [int(s.instance_id), int(s.sample_index), _seg(s), REASON.get(s.finish_reason, -1),
           -1 if s.complete_version is None else int(s.complete_version)]
    if with_tokens:
        rec.append([int(t) for t in s.token_ids()])
        rec.append([float(x) for x in s.behavior_logprob_trace()])
    return rec


def step_record(sched, out, events, with_tokens=False):
    """events: list of [iteration_index, iid, sidx, tokens, reason_str]."""
    buf = sched.buffer
    return {
        "step": int(out.step),
        "batch": [[int(g.instance_id), [int(x) for x in g.completion_seq]] for g in out.batch],
        "samples": [sample_record(s, with_tokens) for g in out.batch for s in g.samples],
        "tokens_generated": int(out.tokens_generated),
        "carried_in_tokens": int(out.carried_in_tokens),
        "groups_completed": int(out.groups_completed),
        "buffer_size_after": int(out.buffer_size_after),
        "pool_size_after": int(out.pool_size_after),
        "open_group_count": int(out.open_group_count),
        "admission": [[KIND[k]] + _sid(sid) for k, sid in out.admission_log],
        "events": [[int(e[0]), int(e[1]), int(e[2]), int(e[3]), REASON[e[4]]] for e in events],
        "partials": [[int(s.instance_id), int(s.sample_index), [int(x) for x in s.paused_at], int(s.total_tokens),
                      _seg(s)] for s in buf.partials()],
        "buffer_ids": [_sid(x) for x in buf.sample_ids()],
        "pool": [[int(s.instance_id), int(s.sample_index), int(s.total_tokens)] for s in sched.pending_pool],
        "iteration_index": int(sched.engine.iteration_index),
        "cumulative_tokens": int(sched.engine.cumulative_tokens),
        "high_water": int(buf.high_water),
    }


def digest(rec) -> str:
    blob = json.dumps(rec, sort_keys=True, separators=(",", ":")).encode()
    return hashlib.sha256(blob).hexdigest()


def first_diff(a, b, path=""):
    """Human-readable first difference between two records (for assertion messages)."""
    if type(a) != type(b):
        return f"{path}: type {type(a).__name__} != {type(b).__name__}"
    if isinstance(a, dict):
        for k in sorted(set(a) | set(b)):
            if k not in a or k not in b:
                return f"{path}.{k}: missing on one side"
            d = first_diff(a[k], b[k], f"{path}.{k}")
            if d:
                return d
        return None
    if isinstance(a, list):
        for i, (x, y) in enumerate(zip(a, b)):
            d = first_diff(x, y, f"{path}[{i}]")
            if d:
                return d
        if len(a) != len(b):
            return f"{path}: len {len(a)} != {len(b)}"
        return None
    return None if a == b else f"{path}: {a!r} != {b!r}"
