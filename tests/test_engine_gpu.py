"""Engine and scheduler known-answer tests on the GPU engine.

Adapted from the reference suite (tests/test_engine.py, tests/test_scheduler.py
of the reference pkg); clock assertions become iteration/token assertions
because the B200 clock is measured wall time, not the d0 + d1*b model.
"""

import numpy as np
import pytest

import paper_2509_18521_b200 as pb
from paper_2509_18521_b200.rollouts import MAX_LENGTH, PAUSED, PENDING, TARGET_LENGTH, RolloutSample

pytestmark = pytest.mark.gpu


def _sample(iid, sidx=0, target=None):
    s = RolloutSample(iid, sidx)
    s.target_length = target
    return s


def _engine(slots=8, l_max=1000):
    eng = pb.LengthDrivenEngine(pb.EngineConfig(max_slots=slots, l_max=l_max), max_handles=256)
    eng.begin_step(0)
    return eng


def test_submit_admits_at_next_boundary():  # reference tests/test_engine.py:32-37
    eng = _engine(slots=4)
    eng.submit(_sample(0, target=5))
    assert eng.active_count == 0
    eng.decode_iteration()
    assert eng.active_count == 1


def test_overflow_queues_fifo():  # :40-47
    eng = _engine(slots=4)
    for i in range(5):
        eng.submit(_sample(i, target=50))
    eng.decode_iteration()
    assert eng.active_count == 4 and eng.queued_count == 1
    assert [s.instance_id for s in eng.active_samples()] == [0, 1, 2, 3]


def test_identical_batch_iterations_and_tokens():  # :50-64
    eng = _engine(slots=8)
    for i in range(6):
        eng.submit(_sample(i, target=40))
    events = []
    while True:
        evs = eng.decode_until_event()
        if not evs:
            break
        events += evs
    assert eng.iteration_index == 40 and eng.cumulative_tokens == 240
    assert len(events) == 6 and all(e.reason == TARGET_LENGTH for e in events)


def test_token_conservation_at_every_boundary():  # :73-84
    rng = np.random.default_rng(0)
    eng = _engine(slots=5, l_max=60)
    samples = [_sample(i, target=int(rng.integers(1, 60))) for i in range(12)]
    for s in samples:
        eng.submit(s)
    while True:
        evs = eng.decode_iteration()
        assert eng.cumulative_tokens == sum(s.total_tokens for s in samples)
        if not evs and eng.idle:
            break


def test_abort_preserves_token_counts():  # :87-101
    eng = _engine(slots=4)
    for i in range(3):
        eng.submit(_sample(i, target=500))
    for _ in range(100):
        eng.decode_iteration()
    back = eng.abort_active()
    assert [s.total_tokens for s in back] == [100, 100, 100]
    assert all(s.status == PAUSED for s in back) and eng.idle
    it = eng.iteration_index
    assert eng.abort_active() == [] and eng.iteration_index == it


def test_abort_drains_queue_as_pending():  # :104-113
    eng = _engine(slots=2)
    for i in range(4):
        eng.submit(_sample(i, target=50))
    eng.decode_iteration()
    back = eng.abort_active()
    st = {s.instance_id: s.status for s in back}
    assert st[0] == st[1] == PAUSED and st[2] == st[3] == PENDING
    assert back[2].total_tokens == 0


def test_submit_completed_sample_is_rejected():  # :116-123
    eng = _engine()
    s = _sample(0, target=1)
    eng.submit(s)
    eng.decode_iteration()
    assert s.status == "completed"
    with pytest.raises(pb.ContractViolation):
        eng.submit(s)


def test_resume_segments_137_363():  # :126-150
    eng = _engine(slots=2)
    s = _sample(0, target=500)
    eng.submit(s)
    for _ in range(137):
        eng.decode_iteration()
    (p,) = eng.abort_active()
    assert p.total_tokens == 137
    eng.begin_step(1)
    eng.submit(p)
    while not eng.idle:
        eng.decode_until_event()
    assert s.total_tokens == 500
    assert [g.token_count for g in s.segments] == [137, 363]
    assert [g.version for g in s.segments] == [0, 1]
    assert s.finish_reason == TARGET_LENGTH


def test_length_cap_reason():  # :153-160
    eng = _engine(l_max=50)
    s = _sample(0, target=5000)
    eng.submit(s)
    while not eng.idle:
        eng.decode_until_event()
    assert s.total_tokens == 50 and s.finish_reason == MAX_LENGTH


def test_event_jump_equals_single_iterations():  # :163-187
    def run(step):
        rng = np.random.default_rng(42)
        eng = _engine(slots=3, l_max=40)
        for i in range(9):
            eng.submit(_sample(i, target=int(rng.integers(1, 40))))
        trace = []
        while True:
            trace += [(e.iteration, e.sample_id, e.tokens, e.reason) for e in step(eng)]
            if eng.idle:
                break
        return trace, eng.iteration_index, eng.cumulative_tokens

    assert run(pb.LengthDrivenEngine.decode_iteration) == run(pb.LengthDrivenEngine.decode_until_event)


def test_same_version_resume_is_a_contract_violation():
    eng = _engine(slots=2)
    s = _sample(0, target=50)
    eng.submit(s)
    eng.decode_iteration()
    (p,) = eng.abort_active()
    eng.submit(p)  # same step: the reference raises at admission (rollouts.py:168-173)
    with pytest.raises(pb.ContractViolation):
        eng.decode_iteration()


def test_begin_step_requires_idle():
    eng = _engine(slots=2)
    eng.submit(_sample(0, target=5))
    with pytest.raises(pb.ContractViolation):
        eng.begin_step(1)


def test_policy_engine_needs_params():  # :238-241
    eng = pb.PolicyDrivenEngine(pb.EngineConfig(max_slots=2, l_max=8), global_seed=0)
    with pytest.raises(pb.ContractViolation):
        eng.begin_step(0, None)


# -- scheduler known answers (reference tests/test_scheduler.py) ------------------------------


def _sched(n=2, g=2, n_prime=4, mode="april", slots=16, l_max=1000, dist=None, seed=0, rho=0.0):
    eng = pb.LengthDrivenEngine(pb.EngineConfig(max_slots=slots, l_max=l_max), max_handles=512)
    cfg = pb.SchedulerConfig(rollout_batch_size=n, samples_per_prompt=g, over_sampling_batch_size=n_prime, mode=mode)
    dist = dist or pb.LengthDistribution.constant(100, l_max)
    return pb.Scheduler(cfg, eng, pb.InstanceSource(group_size=g), pb.LengthSampler(dist, rho, seed))


def _paused(iid, sidx, tokens, version, sched):  # reference tests/test_scheduler.py:43-57
    s = RolloutSample(iid, sidx)
    s.target_length = tokens + 50
    seg = s.open_segment(version, with_tokens=False)
    seg.token_count = tokens
    s.status = PAUSED
    s.paused_at = (version, 0, iid, sidx)
    grp = sched._carryover.get(iid)
    if grp is None:
        grp = pb.Group(pb.PromptInstance(iid, "t", sched.config.samples_per_prompt), [])
        sched._carryover[iid] = grp
    grp.samples.append(s)
    sched.buffer.push_partials([s])
    return s


def test_surplus_groups_delivered_first_next_step():  # :197-209
    sched = _sched()
    o1 = sched.run_step_april(0)
    assert [g.instance_id for g in o1.batch] == [0, 1] and o1.buffer_size_after == 4
    o2 = sched.run_step_april(1)
    assert [g.instance_id for g in o2.batch] == [2, 3]
    assert o2.tokens_generated == 0 and o2.carried_in_tokens == 400 and o2.buffer_size_after == 0


def test_resume_is_fifo_by_pause_time():  # :215-222
    sched = _sched(n_prime=8)
    for step, iid in [(3, 30), (4, 40), (5, 50)]:
        _paused(iid, 0, 20, step, sched)
    assert sched.resume_from_buffer(version=6) == 3
    assert [s.instance_id for s in sched.engine._queue] == [30, 40, 50]


def test_resume_respects_group_capacity():  # :230-237
    sched = _sched(n=1, g=1, n_prime=2)
    for step, iid in [(1, 10), (2, 20), (3, 30)]:
        _paused(iid, 0, 10, step, sched)
    assert sched.resume_from_buffer(version=4) == 2
    assert [s.instance_id for s in sched.buffer.partials()] == [30]


def test_zero_token_samples_return_to_pool():  # :268-285
    sched = _sched(n=1, g=4, n_prime=2, slots=2)
    for j in range(4):
        _paused(500, j, 95, 0, sched)
    out = sched.run_step_april(1)
    assert [g.instance_id for g in out.batch] == [500] and out.pool_size_after > 0
    for s in sched.pending_pool:
        assert s.total_tokens == 0 and s.status == "pending" and not s.segments
    out2 = sched.run_step_april(2)
    assert "pooled" in {k for k, _ in out2.admission_log}


def test_exactly_once_delivery_over_long_run():  # :178-192
    sched = _sched(n=4, g=3, n_prime=8, slots=24, l_max=600, dist=pb.LengthDistribution.lognormal(4.5, 1.1, 600),
                   seed=7)
    seen = set()
    for k in range(120):
        ids = [s.sample_id for s in sched.run_step_april(k).batch_samples()]
        assert len(ids) == 12 and not seen.intersection(ids)
        seen.update(ids)
    left = sched.undelivered_sample_ids()
    assert len(left) == len(set(left)) and not seen.intersection(left)
    assert sched.created_samples == len(seen) + len(left)


def test_group_advantages_kernel_matches_numpy():
    rng = np.random.default_rng(1)
    for g in (1, 2, 7, 8, 16, 33, 64, 65, 129, 200, 1500):  # > 128: numpy's recursive pairwise blocks
        r = rng.random(g * 11)
        for mode in ("mean_baseline", "mean_std_baseline"):
            a = pb.batch_advantages(r, g, mode, 1e-6)
            ref = []
            for k in range(11):
                x = r[k * g:(k + 1) * g]
                c = x - x.mean()
                ref.append(c if mode == "mean_baseline" else c / (x.std() + 1e-6))
            assert np.array_equal(a, np.concatenate(ref)), (g, mode)
    a, flags = pb.batch_advantages(np.array([0.5] * 8 + [0.0, 1.0] * 4), 8, "dapo", return_flags=True)
    assert flags.tolist() == [1, 0]
    # GSPO normalises like GRPO (its sequence ratio comes from Engine.sequence_logprobs)
    r = rng.random(8 * 5)
    assert np.array_equal(pb.batch_advantages(r, 8, "gspo"), pb.batch_advantages(r, 8, "mean_std_baseline"))


def test_clipped_ratio_kernel_matches_oracle():
    """K7 (trainer-side consumption) against the CPU restatement of the reference's clip
    rule (oracle/trainer_ref.py; src/april_sim/policy.py:153-177): ratios and clip masks exact up to
    exp's last ulp, surrogate sums within 1e-12 relative (warp-tree vs numpy summation order)."""
    from oracle import trainer_ref

    rng = np.random.default_rng(3)
    lens = [0, 1, 5, 31, 32, 33, 700, 4096]
    beh = [np.log(rng.uniform(1e-4, 1.0, n)) for n in lens]
    now = [b + rng.normal(0.0, 0.3, b.size) for b in beh]
    adv = rng.normal(0.0, 1.0, len(lens))
    adv[2] = 0.0
    for seq in (False, True):
        r, m, tot = pb.clipped_ratio_terms(now, beh, adv, 0.2, 0.28, sequence_level=seq)
        rr, mr, sr = trainer_ref.clipped_ratio_terms(now, beh, adv, 0.2, 0.28, sequence_level=seq)
        for a, b, ma, mb in zip(r, rr, m, mr):
            np.testing.assert_allclose(a, b, rtol=4e-16, atol=0)
            assert np.array_equal(ma, mb)
        assert abs(tot - sum(sr)) <= 1e-12 * max(1.0, sum(abs(x) for x in sr))
    # identical policies: every ratio is 1 and nothing is clipped
    r, m, _ = pb.clipped_ratio_terms(beh, beh, adv)
    assert all(np.all(x == 1.0) for x in r) and not any(np.any(x) for x in m)
    with pytest.raises(pb.ContractViolation):
        pb.clipped_ratio_terms(now[:2], beh[:2][::-1], adv[:2])


def test_out_of_kv_fails_without_leaking_pages():
    """a failed page pop must leave the free-page stack intact.  A prompt group that does
    not fit raises OutOfKV; releasing what it got restores the pool exactly, and decoding that
    exhausts the pool mid-iteration stops with OutOfKV, the top never negative."""
    from paper_2509_18521_b200 import _capi

    spec = pb.PRESETS["tiny"]
    prompts = {i: pb.synthetic_prompt(2, i, 100, spec.vocab) for i in range(8)}
    eng = pb.LengthDrivenEngine(pb.EngineConfig(max_slots=8, l_max=512), model=spec, prompt_len=100,
                                page_size=16, kv_pages=10, max_handles=32, max_groups=8,
                                prompt_source=lambda iid: prompts[iid])
    total = eng.stats().kv_pages_free
    assert total == 10
    eng.begin_step(0)
    a = _sample(0, 0, 40)
    eng.submit(a)  # group 0: 99 prompt positions -> 7 pages, the sample's tail page copy -> 1 page
    eng._flush()
    assert eng.stats().kv_pages_free == 10 - 8
    b = _sample(1, 0, 40)
    with pytest.raises(_capi.OutOfKV):  # group 1 needs 7 more pages, 2 are left
        eng.submit(b)
        eng._flush()
    # the failed prefill returned its partial allocation: the 2 free pages are free again
    assert eng.stats().kv_pages_free == 2
    eng._queue.remove(b)
    eng._release([b])
    assert eng.stats().kv_pages_free == 2
    while not eng.idle:  # the first sample still fits: 40 tokens from position 99 need 2 new pages
        eng.decode_until_event()
    assert a.total_tokens == 40
    assert eng.stats().kv_pages_free == total  # everything went back
    eng.close()
    # decode exhaustion: two samples growing past the pool
    eng = pb.LengthDrivenEngine(pb.EngineConfig(max_slots=8, l_max=512), model=spec, prompt_len=100,
                                page_size=16, kv_pages=12, max_handles=32, max_groups=8,
                                prompt_source=lambda iid: prompts[iid])
    eng.begin_step(0)
    for j in range(2):
        eng.submit(_sample(0, j, 400))
    with pytest.raises(_capi.OutOfKV):
        while not eng.idle:
            eng.decode_until_event()
    free = eng.stats().kv_pages_free
    assert 0 <= free < 2, free
    eng.close()
