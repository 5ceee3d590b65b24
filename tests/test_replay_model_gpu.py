"""Bit-exact replay with the transformer ON: the bench's code path against the reference goldens.

In length-trace replay mode (north star) every scheduling, abort and recycle decision and the
buffer contents must equal the reference's, whatever tokens the model samples: the trace decides
when a sample stops.  `tests/test_replay_gpu.py` checks that with the model off; here every
iteration is a real decode step (tcgen05 GEMMs, paged attention, fused sampler) and the stop rule is
the sampler epilogue's copy of the trace stop (`csrc/sampler.cu`), with KV pages allocated during
admission, the reduce-added split-K GEMMs of the bench (`nondeterministic_gemm`), and both KV resume
modes (`retain`, and `reprefill`: the abort drops a partial's KV, the resubmit re-prefills it).

Reference: src/april_sim/engine.py:167-180 (advance), :220-240 (trace stop),
src/april_sim/scheduler.py:232-393 (the APRIL step); goldens from tests/golden/make_goldens.py.
"""

import pytest

import canon
import goldens
import paper_2509_18521_b200 as pb
from product_runs import make_scheduler, product_replay

pytestmark = pytest.mark.gpu


def _strip(r):
    return {k: v for k, v in r.items() if k != "rollout_wall_time"}


def _model_kw(spec, kv_resume, nondet, temperature=0.8):
    return dict(model=spec, sampling=pb.SamplingConfig(temperature=temperature), prompt_len=64,
                page_size=64 if spec.vocab > 4096 else 16, kv_resume=kv_resume, nondeterministic_gemm=nondet)


@pytest.mark.parametrize("kv_resume", ["retain", "reprefill"])
@pytest.mark.parametrize("nondet", [False, True])
@pytest.mark.parametrize("mode", ["april", "baseline"])
def test_c1_tiny_model_replay_matches_reference(mode, nondet, kv_resume):
    g = goldens.replay("C1", mode)
    recs, sched = product_replay(canon.CONFIGS["C1"], mode, len(g["records"]),
                                 **_model_kw(pb.PRESETS["tiny"], kv_resume, nondet))
    for k, (mine, ref) in enumerate(zip(recs, g["records"])):
        assert mine == _strip(ref), f"step {k}: " + str(canon.first_diff(mine, _strip(ref)))
    eng = sched.engine
    st = eng.stats()
    # every page not held by a resident group or a parked partial went back to the pool
    assert st.kv_pages_free <= st.kv_pages_total
    eng.close()


@pytest.mark.parametrize("kv_resume", ["retain", "reprefill"])
def test_c2_shape_model_replay_matches_reference_digests(kv_resume):
    """C2 (S = 1024, l_max 4096, 6 APRIL steps) with the Qwen2.5-1.5B shape cut to 2 layers."""
    dg = goldens.digests()["C2/april"]
    spec = pb.PRESETS["qwen2.5-1.5b"].truncated(2)
    recs, sched = product_replay(canon.CONFIGS["C2"], "april", len(dg), **_model_kw(spec, kv_resume, True))
    assert [canon.digest(r) for r in recs] == dg
    sched.engine.close()


def test_c2_shape_model_sync_replay_matches_reference_digests():
    dg = goldens.digests()["C2/baseline"]
    spec = pb.PRESETS["qwen2.5-1.5b"].truncated(2)
    recs, sched = product_replay(canon.CONFIGS["C2"], "baseline", len(dg), **_model_kw(spec, "reprefill", True))
    assert [canon.digest(r) for r in recs] == dg
    sched.engine.close()


def test_c3_shape_model_replay_matches_reference():
    """C3 (S = 64, l_max 16384: contexts past 16k, multi-split attention rows, DAPO-sized groups) with
    the Qwen3-4B shape cut to 1 layer, KV re-prefill on, full canonical records."""
    g = goldens.replay("C3", "april")
    spec = pb.PRESETS["qwen3-4b"].truncated(1)
    recs, sched = product_replay(canon.CONFIGS["C3"], "april", len(g["records"]),
                                 **_model_kw(spec, "reprefill", True))
    for k, (mine, ref) in enumerate(zip(recs, g["records"])):
        assert mine == _strip(ref), f"step {k}: " + str(canon.first_diff(mine, _strip(ref)))
    sched.engine.close()


def test_model_on_delivered_payload_matches_token_counts():
    """The device payload read back at delivery has one token id and one finite log-prob per token,
    including samples resumed across steps (re-prefilled KV) whose payload spans several segments."""
    import math

    spec = pb.PRESETS["tiny"]
    sched = make_scheduler(canon.CONFIGS["C1"], "april", **_model_kw(spec, "reprefill", True))
    multi = 0
    for k in range(6):
        out = sched.run_step(k)
        for s in out.batch_samples():
            toks, lps = s.token_ids(), s.behavior_logprob_trace()
            assert len(toks) == len(lps) == s.total_tokens
            assert all(0 <= t < spec.vocab for t in toks)
            assert all(math.isfinite(x) and x <= 0 for x in lps)
            multi += len(s.segments) > 1
    assert multi > 0, "no delivered sample spanned a resume"
    sched.engine.close()


@pytest.mark.parametrize("name,preset,layers", [("C4_1.5", "qwen3-4b", 1), ("C4_3", "qwen3-4b", 1),
                                                ("C5", "r1-distill-7b", 1)])
def test_c4_c5_shape_model_replay_matches_reference_digests(name, preset, layers):
    """C4 (GSPO-sized heavy tail, L_max 16384, N'/N = 1.5 and 3 at S = 64: the queued surplus returns
    to the pool) and C5 (256 x 16 samples per step at S = 1024; untied lm_head, GQA 7:1, QKV bias) with
    the model ON (depth cut so the reference config's KV fits one GPU); trace mode, so the decisions
    must equal the reference goldens' digests."""
    dg = goldens.digests()[f"{name}/april"]
    spec = pb.PRESETS[preset].truncated(layers)
    recs, sched = product_replay(canon.CONFIGS[name], "april", len(dg), **_model_kw(spec, "reprefill", True))
    assert [canon.digest(r) for r in recs] == dg
    sched.engine.close()


@pytest.mark.parametrize("name", ["C4_3", "C3"])
def test_kv_pages_conserved_across_steps(name):
    """KV page conservation with the bench's re-prefill mode at S = 64 and a long partial buffer: after
    each step's abort the pages in use are exactly the resident prompt groups' pages plus one private
    tail page per held sample that has not generated a token (its fork), nothing else."""
    spec = pb.PRESETS["qwen3-4b"].truncated(1)
    cfg = canon.CONFIGS[name]
    sched = make_scheduler(cfg, "april", **_model_kw(spec, "reprefill", True))
    eng = sched.engine
    P, prompt = eng.page_size, eng.prompt_len
    per_group = (prompt - 1 + P - 1) // P
    tail = 1 if (prompt - 1) % P else 0
    for k in range(4):
        sched.run_step(k)
        st = eng.stats()
        used = st.kv_pages_total - st.kv_pages_free
        held_zero = sum(1 for h, s in eng._by_handle.items() if s.total_tokens == 0)
        expect = per_group * len(eng._gslot) + tail * held_zero
        assert used == expect, (k, used, expect, len(eng._gslot), held_zero, len(eng._by_handle))
    eng.close()
