"""Transformer decode path on the GPU vs the torch-CPU oracle (oracle/cpu_model.py).

Greedy decoding: every generated token must be the oracle's argmax given the
same prefix (teacher-forced), except where the oracle's own top-2 margin is
below MARGIN_EPS (a near-tie that bf16 rounding may legitimately flip; such
positions are counted and bounded).  Log-probs must agree within LOGP_TOL.
"""

import numpy as np
import pytest

import paper_2509_18521_b200 as pb
from paper_2509_18521_b200.rollouts import RolloutSample

torch = pytest.importorskip("torch")
from oracle import rng_ref  # noqa: E402
from oracle.cpu_model import CpuDecoder  # noqa: E402

pytestmark = pytest.mark.gpu

MARGIN_EPS = 0.05   # logit units
LOGP_TOL = 0.05     # nats


def _engine(spec, prompts, S=8, l_max=64, page=16, greedy=True, temperature=1.0, P=None, nondet=False,
            kv_resume="retain", top_p=1.0):
    P = P or max(len(p) for p in prompts.values())
    return pb.LengthDrivenEngine(
        pb.EngineConfig(max_slots=S, l_max=l_max), global_seed=3, model=spec,
        sampling=pb.SamplingConfig(temperature=temperature, greedy=greedy, top_p=top_p), prompt_len=P, page_size=page,
        kv_pages=1024, max_handles=64, max_groups=16, prompt_source=lambda iid: prompts[iid],
        nondeterministic_gemm=nondet, kv_resume=kv_resume)


def _prompts(spec, n, P):
    return {i: pb.synthetic_prompt(11, i, P, spec.vocab) for i in range(n)}


def _drain(eng):
    while not eng.idle:
        eng.decode_until_event()


def _check_greedy(dec, prompt, toks, logps):
    sc = dec.score([int(t) for t in prompt], toks)
    flips = 0
    for k, (t, lp, r) in enumerate(zip(toks, logps, sc)):
        if r["argmax"] != t:
            flips += 1
            assert r["margin"] < MARGIN_EPS, (k, r)
        assert abs(lp - r["logp"]) < LOGP_TOL, (k, lp, r)
    return flips


@pytest.mark.parametrize("nondet", [False, True])
@pytest.mark.parametrize("preset,layers", [("tiny", None), ("qwen2.5-1.5b", 2), ("qwen3-4b", 1)])
def test_greedy_tokens_match_oracle(preset, layers, nondet):
    spec = pb.PRESETS[preset]
    if layers:
        spec = spec.truncated(layers)
    prompts = _prompts(spec, 2, 24)
    eng = _engine(spec, prompts, page=16 if preset == "tiny" else 64, nondet=nondet)
    eng.begin_step(0)
    samples = []
    for iid, lens in ((0, [5, 17, 30, 40]), (1, [9, 33])):
        for j, L in enumerate(lens):
            s = RolloutSample(iid, j)
            s.target_length = L
            eng.submit(s)
            samples.append(s)
    _drain(eng)
    dec = CpuDecoder(spec, eng.export_weights())
    flips = total = 0
    for s in samples:
        assert s.total_tokens == s.target_length and len(s.token_ids()) == s.target_length
    # greedy + shared prompt: all samples of a group generate the same sequence, so
    # the longest one is scored against the oracle and the others must be its prefixes
    # (deterministic schedules only: with reduce-added split-K the rows of one batch may sum
    # their K splits in different orders, so each sample is scored against the oracle instead)
    for iid in (0, 1):
        grp = [s for s in samples if s.instance_id == iid]
        top = max(grp, key=lambda s: s.total_tokens)
        if nondet:
            for s in grp:
                flips += _check_greedy(dec, prompts[iid], s.token_ids(), s.behavior_logprob_trace())
                total += s.total_tokens
            continue
        for s in grp:
            assert s.token_ids() == top.token_ids()[: s.total_tokens]
            np.testing.assert_allclose(s.behavior_logprob_trace(), top.behavior_logprob_trace()[: s.total_tokens],
                                       rtol=0, atol=1e-5)
        flips += _check_greedy(dec, prompts[iid], top.token_ids(), top.behavior_logprob_trace())
        total += top.total_tokens
    # every flip was already checked to be an oracle near-tie (margin < MARGIN_EPS); random-init
    # logits over a 152k vocabulary have many of those, so only bound the rate loosely
    assert flips <= max(3, total // 10), f"{flips} near-tie flips over {total} tokens"
    eng.close()


def test_resume_across_steps_keeps_kv_and_matches_uninterrupted():
    spec = pb.PRESETS["tiny"]
    prompts = _prompts(spec, 1, 20)
    eng = _engine(spec, prompts)
    eng.begin_step(0)
    s = RolloutSample(0, 0)
    s.target_length = 50
    eng.submit(s)
    for _ in range(13):
        eng.decode_iteration()
    (p,) = eng.abort_active()
    assert p.total_tokens == 13
    eng.begin_step(1)
    eng.submit(p)
    _drain(eng)
    assert [g.token_count for g in s.segments] == [13, 37]
    dec = CpuDecoder(spec, eng.export_weights())
    flips = _check_greedy(dec, prompts[0], s.token_ids(), s.behavior_logprob_trace())
    assert flips <= 1
    # identical to an uninterrupted run
    eng2 = _engine(spec, prompts)
    eng2.begin_step(0)
    r = RolloutSample(0, 0)
    r.target_length = 50
    eng2.submit(r)
    _drain(eng2)
    assert r.token_ids() == s.token_ids()
    np.testing.assert_allclose(r.behavior_logprob_trace(), s.behavior_logprob_trace(), rtol=0, atol=1e-6)


def test_nucleus_sampling_in_the_engine():
    """top_p < 1 in the engine's decode loop (K1 nucleus kernel, one CTA per row): every token lies in
    the oracle's nucleus (sampler_ref.nucleus_threshold on the oracle's logits; a token within 1e-3 of
    the threshold is tolerated) and its behaviour logp is the truncated distribution's."""
    from oracle import sampler_ref

    spec = pb.PRESETS["tiny"]
    prompts = _prompts(spec, 1, 16)
    T, top_p = 0.8, 0.9
    eng = _engine(spec, prompts, greedy=False, temperature=T, top_p=top_p)
    eng.begin_step(0)
    s = RolloutSample(0, 1)
    s.target_length = 40
    eng.submit(s)
    _drain(eng)
    toks, lps = s.token_ids(), s.behavior_logprob_trace()
    dec = CpuDecoder(spec, eng.export_weights())
    cache = dec.new_cache()
    prompt = [int(t) for t in prompts[0]]
    dec.forward(prompt[:-1], cache, 0, want_logits=False)
    tok, pos, outside = prompt[-1], len(prompt) - 1, 0
    for k, g in enumerate(toks):
        z = dec.forward([tok], cache, pos).float().numpy()
        kmin = sampler_ref.nucleus_threshold(z, T, top_p)
        keys = sampler_ref.logit_keys(z)
        keep = keys >= np.uint32(kmin)
        if not keep[g]:
            zk = z[keep]
            outside += int(z[g] < zk.min() - 1e-3)
        p = np.exp2((z - z.max()) * np.float32(1.0 / T) * np.float32(1.4426950408889634)).astype(np.float64)
        pk = np.where(keep, p, 0.0)
        ref_lp = float(np.log(p[g] / pk.sum())) if keep[g] else None
        if ref_lp is not None:
            assert abs(lps[k] - ref_lp) < LOGP_TOL, (k, lps[k], ref_lp)
        tok, pos = g, pos + 1
    assert outside == 0


def test_temperature_sampling_follows_philox_inverse_cdf():
    spec = pb.PRESETS["tiny"]
    prompts = _prompts(spec, 1, 16)
    T = 0.8
    eng = _engine(spec, prompts, greedy=False, temperature=T)
    eng.begin_step(0)
    s = RolloutSample(0, 2)
    s.target_length = 40
    eng.submit(s)
    _drain(eng)
    toks, lps = s.token_ids(), s.behavior_logprob_trace()
    dec = CpuDecoder(spec, eng.export_weights())
    key = rng_ref.stream_key(3, rng_ref.LANE_POLICY_TOKENS, 0, 2)
    cache = dec.new_cache()
    prompt = [int(t) for t in prompts[0]]
    dec.forward(prompt[:-1], cache, 0, want_logits=False)
    tok, pos, bad = prompt[-1], len(prompt) - 1, 0
    for k, g in enumerate(toks):
        z = dec.forward([tok], cache, pos)
        p = torch.softmax(z.double() / T, -1)
        cdf = torch.cumsum(p, 0)
        u = rng_ref.raw_uniform(key, k)
        lo = float(cdf[g - 1]) if g > 0 else 0.0
        hi = float(cdf[g])
        if not (lo - 1e-3 <= u <= hi + 1e-3):
            bad += 1
        assert abs(lps[k] - float(torch.log(p[g]))) < LOGP_TOL
        tok, pos = g, pos + 1
    assert bad == 0


def test_kv_pages_are_recycled():
    spec = pb.PRESETS["tiny"]
    prompts = _prompts(spec, 4, 20)
    eng = _engine(spec, prompts)
    free0 = eng.stats().kv_pages_free
    for step in range(3):
        eng.begin_step(step)
        for iid in range(4):
            for j in range(2):
                s = RolloutSample(iid + 10 * step, j)
                s.target_length = 10 + 7 * j
                prompts[iid + 10 * step] = prompts[iid]
                eng.submit(s)
        _drain(eng)
    assert eng.stats().kv_pages_free == free0


def test_sequence_logprobs_reduce_the_resident_payload():
    """GSPO's length-normalised sequence log-prob, reduced on the device while the samples are
    still resident, equals the host sum of the behaviour log-probs delivered later."""
    spec = pb.PRESETS["tiny"]
    prompts = _prompts(spec, 1, 16)
    eng = _engine(spec, prompts, greedy=False, temperature=0.9)
    eng.begin_step(0)
    samples = []
    for j in range(4):
        s = RolloutSample(0, j)
        s.target_length = 30 + j
        eng.submit(s)
        samples.append(s)
    for _ in range(12):
        eng.decode_iteration()
    sums, lens = eng.sequence_logprobs(samples)
    assert lens.tolist() == [12] * 4
    _drain(eng)
    for s, sm, n in zip(samples, sums, lens):
        full = s.behavior_logprob_trace()
        assert len(full) == s.target_length
        assert abs(sm - float(np.sum(full[:n]))) < 1e-9 * max(1.0, abs(sm))
    eng.close()


@pytest.mark.parametrize("preset,layers,page", [("tiny", None, 16), ("qwen2.5-1.5b", 2, 64), ("qwen3-4b", 1, 16)])
def test_long_prompt_prefill_matches_oracle(preset, layers, page):
    """Prompt prefill through the flash prefill kernel: several 64-row blocks per prompt, prompts
    of different lengths packed in one chunk, pages of 16 and 64 tokens."""
    spec = pb.PRESETS[preset]
    if layers:
        spec = spec.truncated(layers)
    prompts = {0: pb.synthetic_prompt(11, 0, 203, spec.vocab), 1: pb.synthetic_prompt(11, 1, 77, spec.vocab)}
    eng = _engine(spec, prompts, page=page, l_max=256)
    eng.begin_step(0)
    samples = []
    for iid in (0, 1):
        s = RolloutSample(iid, 0)
        s.target_length = 12
        eng.submit(s)
        samples.append(s)
    _drain(eng)
    dec = CpuDecoder(spec, eng.export_weights())
    flips = sum(_check_greedy(dec, prompts[s.instance_id], s.token_ids(), s.behavior_logprob_trace())
                for s in samples)
    assert flips <= 2
    eng.close()


@pytest.mark.parametrize("preset,layers,page", [("tiny", None, 16), ("qwen2.5-1.5b", 2, 64), ("qwen3-4b", 1, 16)])
def test_reprefill_resume_matches_oracle(preset, layers, page):
    """KV re-prefill mode: the abort drops the paused samples' KV, the resubmit
    rebuilds it by prefill (prompt tail + carried tokens), and decoding continues on it.  Tokens
    after the resume are checked against the oracle teacher-forced on the full history."""
    spec = pb.PRESETS[preset]
    if layers:
        spec = spec.truncated(layers)
    prompts = _prompts(spec, 2, 37)
    eng = _engine(spec, prompts, page=page, l_max=200, kv_resume="reprefill")
    free0 = eng.stats().kv_pages_free
    eng.begin_step(0)
    samples = []
    for iid in (0, 1):
        for j in range(2):
            s = RolloutSample(iid, j)
            s.target_length = 90 + 17 * j + 5 * iid
            eng.submit(s)
            samples.append(s)
    for _ in range(70):
        eng.decode_iteration()
    paused = eng.abort_active()
    assert len(paused) == 4 and all(p.total_tokens == 70 for p in paused)
    pf0 = eng.stats().prefill_tokens
    eng.begin_step(1)  # new version: the resident groups' prompt KV is recomputed in place
    for p in paused:
        eng.submit(p)
    _drain(eng)
    assert eng.stats().prefill_tokens == pf0 + 2 * 36
    st = eng.stats()
    assert st.reprefill_tokens == 4 * 70
    dec = CpuDecoder(spec, eng.export_weights())
    flips = 0
    for s in samples:
        assert [g.token_count for g in s.segments] == [70, s.target_length - 70]
        flips += _check_greedy(dec, prompts[s.instance_id], s.token_ids(), s.behavior_logprob_trace())
    assert flips <= max(3, sum(s.target_length for s in samples) // 25)
    eng.discard(samples)
    assert eng.stats().kv_pages_free == free0
    eng.close()



@pytest.mark.parametrize("preset,layers", [("tiny", None), ("qwen2.5-1.5b", 2), ("qwen3-4b", 1)])
def test_score_recomputes_behaviour_logprobs(preset, layers):
    """Trainer-side recompute: teacher-forced log-probs of delivered responses under the
    current weights match the oracle's, and (same weights) the behaviour log-probs recorded while
    sampling; one response longer than a page, prompts of different lengths."""
    spec = pb.PRESETS[preset]
    if layers:
        spec = spec.truncated(layers)
    prompts = {0: pb.synthetic_prompt(11, 0, 23, spec.vocab), 1: pb.synthetic_prompt(11, 1, 40, spec.vocab)}
    eng = _engine(spec, prompts, greedy=False, temperature=0.9, l_max=128)
    free0 = eng.stats().kv_pages_free
    eng.begin_step(0)
    samples = []
    for iid, L in ((0, 70), (0, 9), (1, 33)):
        s = RolloutSample(iid, len(samples))
        s.target_length = L
        eng.submit(s)
        samples.append(s)
    _drain(eng)
    now = eng.recompute_logprobs(samples)
    assert eng.stats().kv_pages_free == free0  # the scratch pages went back to the pool
    dec = CpuDecoder(spec, eng.export_weights())
    for s, lp in zip(samples, now):
        beh = np.asarray(s.behavior_logprob_trace())
        assert lp.shape == beh.shape
        assert np.max(np.abs(lp - beh)) < LOGP_TOL
        sc = dec.score([int(t) for t in prompts[s.instance_id]], s.token_ids(), temperature=0.9)
        ref = np.array([r["logp"] for r in sc])
        assert np.max(np.abs(lp - ref)) < LOGP_TOL
    ratios, masks, _ = pb.policy.clipped_ratio_terms(now, [s.behavior_logprob_trace() for s in samples],
                                                     [1.0, -1.0, 0.5])
    assert all(np.all(np.abs(r - 1.0) < 0.06) for r in ratios)
    eng.close()


def test_weight_swap_then_reprefill_resume_follows_new_weights():
    """SURVEY §8 f4 + f1: new policy weights are installed between steps; the resumed partials' KV is
    re-prefilled under them, so every token generated after the resume is the new model's choice given
    the whole (mixed-policy) history.  Checked teacher-forced against the oracle with the new weights."""
    spec = pb.PRESETS["qwen2.5-1.5b"].truncated(2)
    prompts = _prompts(spec, 1, 30)
    eng = _engine(spec, prompts, page=16, l_max=128, kv_resume="reprefill")
    eng.begin_step(0)
    samples = []
    for j in range(2):
        s = RolloutSample(0, j)
        s.target_length = 60 + 5 * j
        eng.submit(s)
        samples.append(s)
    for _ in range(25):
        eng.decode_iteration()
    paused = eng.abort_active()
    w = eng.export_weights()
    g = torch.Generator().manual_seed(7)
    new = {}
    for k, t in w.items():
        if "norm" in k:
            continue
        new[k] = (t.float() + 0.02 * torch.randn(t.shape, generator=g)).to(torch.bfloat16)
    eng.load_weights(new)
    eng.begin_step(1)
    for p in paused:
        eng.submit(p)
    _drain(eng)
    dec = CpuDecoder(spec, eng.export_weights())
    for s in samples:
        toks, lps = s.token_ids(), s.behavior_logprob_trace()
        sc = dec.score([int(t) for t in prompts[0]], toks)
        flips = 0
        for k in range(25, len(toks)):
            if sc[k]["argmax"] != toks[k]:
                flips += 1
                assert sc[k]["margin"] < MARGIN_EPS, (k, sc[k])
            assert abs(lps[k] - sc[k]["logp"]) < LOGP_TOL, (k, lps[k], sc[k])
        assert flips <= 4
    eng.close()


def test_kv_memory_release_and_resume():
    """SURVEY §8 f4 memory hand-off: between steps the KV pool is freed (HBM returns to the device)
    and re-acquired; resident prompt KV is recomputed and the resumed partials are re-prefilled, so
    decoding continues exactly as the model dictates (oracle, teacher-forced)."""
    spec = pb.PRESETS["tiny"]
    prompts = _prompts(spec, 2, 21)
    eng = _engine(spec, prompts, l_max=128, kv_resume="reprefill")
    eng.begin_step(0)
    samples = []
    for iid in (0, 1):
        s = RolloutSample(iid, 0)
        s.target_length = 50 + 7 * iid
        eng.submit(s)
        samples.append(s)
    for _ in range(20):
        eng.decode_iteration()
    paused = eng.abort_active()
    free_before = torch.cuda.mem_get_info()[0]
    eng.release_memory()
    assert torch.cuda.mem_get_info()[0] > free_before  # the pool went back to the device
    with pytest.raises(pb.ContractViolation):
        eng.submit(paused[0])
        eng._flush()
    eng._pending.clear()
    eng._queue.clear()
    eng.resume_memory()
    eng.begin_step(1)
    for p in paused:
        eng.submit(p)
    _drain(eng)
    dec = CpuDecoder(spec, eng.export_weights())
    flips = sum(_check_greedy(dec, prompts[s.instance_id], s.token_ids(), s.behavior_logprob_trace())
                for s in samples)
    assert flips <= 3
    eng.close()
