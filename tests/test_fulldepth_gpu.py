"""Full-depth greedy parity: the bench's models at every layer, long generations.

C2 (Qwen2.5-1.5B shape, 28 layers) and C3 (Qwen3-4B shape, 36 layers) at full depth, 256-token
prompts, rows generating up to 1,600 tokens greedily on the GPU (contexts ~1,850 tokens, several
attention tiles and pages per row, the live batch shrinking as rows finish), then scored
teacher-forced by the fp32 CPU oracle (`oracle/cpu_model.py`, one causal pass over prompt +
response) on the GPU's exported bf16 weights.

Contract.  The oracle fixes where activations are rounded to bf16, not the fp32 summation order
inside a projection, so two correct implementations drift apart at full depth (a bf16 rounding lands
on the other side now and then, and the difference propagates through 28-36 layers).  The test
therefore measures that noise floor on the same weights and tokens: the oracle summing in fp32 vs
the oracle summing in fp64 (`CpuDecoder(compute_dtype=float64)`, same roundings; the fp64 form is
the reference "exact" contract).  Against the fp64 form the GPU must be (stated tolerances):
* flips (GPU token != fp64 argmax) only where the fp64 margin is below MARGIN_EPS logits, and at
  most FLOOR_FACTOR x the fp32 oracle's own flip fraction + 1 %;
* max and mean |behaviour logp - fp64 logp| at most FLOOR_FACTOR x the fp32 oracle's, and the max
  below LOGP_CAP nats (T = 1).
Measured values are written to profiles/r2_fulldepth_*.json (AB_TEST_REPORT_DIR).
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

MARGIN_EPS = 0.1    # logits
FLOOR_FACTOR = 2.5
LOGP_CAP = 0.15     # nats
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
    exact = CpuDecoder(spec, weights, compute_dtype=torch.float64)
    del weights
    report = {"preset": preset, "layers": spec.n_layers, "nondeterministic_gemm": nondet, "rows": []}
    for s in samples:
        toks, lps = s.token_ids(), np.asarray(s.behavior_logprob_trace())
        assert len(toks) == s.target_length
        prompt = [int(t) for t in prompts[s.instance_id]]
        ex = exact.score_all(prompt, toks)
        f32 = dec.score_all(prompt, toks)
        flip = ex["argmax"] != np.asarray(toks)
        d_gpu = np.abs(lps - ex["logp"])
        d_f32 = np.abs(f32["logp"] - ex["logp"])
        row = {"generated": len(toks), "gpu_flips": int(flip.sum()),
               "gpu_max_flip_margin": float(ex["margin"][flip].max()) if flip.any() else 0.0,
               "gpu_max_abs_dlogp": float(d_gpu.max()), "gpu_mean_abs_dlogp": float(d_gpu.mean()),
               "fp32_oracle_flips": int((f32["argmax"] != ex["argmax"]).sum()),
               "fp32_oracle_max_abs_dlogp": float(d_f32.max()), "fp32_oracle_mean_abs_dlogp": float(d_f32.mean()),
               "median_top2_margin": float(np.median(ex["top2"]))}
        report["rows"].append(row)
        print(json.dumps(row))
    out = os.environ.get("AB_TEST_REPORT_DIR")
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, f"fulldepth_{preset}_{'nondet' if nondet else 'det'}.json"), "w") as f:
            json.dump(report, f, indent=1)
    for row in report["rows"]:
        n = row["generated"]
        assert row["gpu_max_flip_margin"] < MARGIN_EPS, row
        assert row["gpu_flips"] <= FLOOR_FACTOR * row["fp32_oracle_flips"] + 0.01 * n, row
        assert row["gpu_max_abs_dlogp"] <= max(FLOOR_FACTOR * row["fp32_oracle_max_abs_dlogp"], 1e-3), row
        assert row["gpu_mean_abs_dlogp"] <= max(FLOOR_FACTOR * row["fp32_oracle_mean_abs_dlogp"], 1e-4), row
        assert row["gpu_max_abs_dlogp"] <= LOGP_CAP, row
