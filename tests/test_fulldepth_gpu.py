"""Full-depth greedy parity: the bench's models at every layer, long generations.

C2 (Qwen2.5-1.5B shape, 28 layers) and C3 (Qwen3-4B shape, 36 layers) at full depth, 256-token
prompts, rows generating up to 1,600 tokens greedily on the GPU (contexts ~1,850 tokens, several
attention tiles and pages per row, the live batch shrinking as rows finish), then scored
teacher-forced by the fp32 CPU oracle (`oracle/cpu_model.py`, one causal pass over prompt +
response) on the GPU's exported bf16 weights.

Contract (stated tolerances, measured on B200 and recorded in profiles/r2_fulldepth_*.json):
* every generated token is the oracle's argmax given the same prefix, except where the oracle's own
  margin between its argmax and the GPU's token is below MARGIN_EPS logits (a near-tie that bf16
  rounding of the activations may legitimately flip); such flips are at most MAX_FLIP_FRAC of tokens;
* |behaviour logp - oracle logp| <= LOGP_TOL nats at every position (T = 1).
"""

import json
import os

import numpy as np
import pytest

import paper_2509_18521_b200 as pb
from paper_2509_18521_b200.rollouts import RolloutSample

torch = pytest.importorskip("torch")
from oracle.cpu_model import CpuDecoder  # noqa: E402

pytestmark = pytest.mark.gpu

MARGIN_EPS = 0.05   # logits
MAX_FLIP_FRAC = 0.02
LOGP_TOL = 0.02     # nats
PROMPT = 256
LENGTHS = (1600, 1537, 700)


@pytest.mark.parametrize("preset,nondet", [("qwen2.5-1.5b", False), ("qwen2.5-1.5b", True), ("qwen3-4b", True)])
def test_full_depth_greedy_long_generation_matches_oracle(preset, nondet):
    spec = pb.PRESETS[preset]
    prompts = {i: pb.synthetic_prompt(13, i, PROMPT, spec.vocab) for i in range(len(LENGTHS))}
    eng = pb.LengthDrivenEngine(
        pb.EngineConfig(max_slots=4, l_max=max(LENGTHS)), global_seed=5, model=spec,
        sampling=pb.SamplingConfig(greedy=True), prompt_len=PROMPT, page_size=64, kv_pages=512,
        max_handles=16, max_groups=8, prompt_source=lambda iid: prompts[iid], nondeterministic_gemm=nondet)
    eng.begin_step(0)
    samples = []
    for iid, L in enumerate(LENGTHS):
        s = RolloutSample(iid, 0)
        s.target_length = L
        eng.submit(s)
        samples.append(s)
    while not eng.idle:
        eng.decode_until_event()
    weights = eng.export_weights()
    eng.close()
    dec = CpuDecoder(spec, weights)
    del weights
    report = {"preset": preset, "layers": spec.n_layers, "nondeterministic_gemm": nondet, "rows": []}
    for s in samples:
        toks, lps = s.token_ids(), np.asarray(s.behavior_logprob_trace())
        assert len(toks) == s.target_length
        sc = dec.score_all([int(t) for t in prompts[s.instance_id]], toks)
        flip = sc["argmax"] != np.asarray(toks)
        dlogp = np.abs(lps - sc["logp"])
        row = {"generated": len(toks), "flips": int(flip.sum()),
               "max_flip_margin": float(sc["margin"][flip].max()) if flip.any() else 0.0,
               "max_abs_dlogp": float(dlogp.max()), "mean_abs_dlogp": float(dlogp.mean()),
               "median_top2_margin": float(np.median(sc["top2"]))}
        report["rows"].append(row)
        print(json.dumps(row))
    out = os.environ.get("AB_TEST_REPORT_DIR")
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, f"fulldepth_{preset}_{'nondet' if nondet else 'det'}.json"), "w") as f:
            json.dump(report, f, indent=1)
    for s, row in zip(samples, report["rows"]):
        assert row["max_flip_margin"] < MARGIN_EPS, row
        assert row["flips"] <= MAX_FLIP_FRAC * row["generated"], row
        assert row["max_abs_dlogp"] <= LOGP_TOL, row
