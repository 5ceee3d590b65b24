"""Pin the transformer oracle (oracle/cpu_model.py) to an independent implementation.

The reference has no model: the decode numerics oracle is the builder's own
restatement, so here it is checked against `transformers`' Qwen2ForCausalLM / Qwen3ForCausalLM
(5.5, in the image) on the same weights, in the engine's export layout (fused QKV rows [q | k | v],
gate/up rows tile-interleaved per 128 rows, bias / q-k-norm / tied or untied embeddings as the
preset has them).  Norm weights and biases are random (not ones / zeros) so their placement is
pinned too.  `CpuDecoder(round_bf16=False)` runs the oracle's math without the engine's bf16
activation roundings; what remains is fp32 summation order: max |delta logit| <= 1e-3 (stated).
This pins RoPE (rotate-half, theta, inv_freq), q/k-norm placement, the GQA head mapping, SwiGLU and
the gate/up un-interleave; the bf16 roundings on top are the engine's documented numerics.
"""

import pytest

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

import paper_2509_18521_b200 as pb  # noqa: E402
from oracle.cpu_model import CpuDecoder, random_weights, split_gate_up  # noqa: E402

TOL = 1e-3


def _spec(kind):
    if kind == "qwen2":  # C2 head layout (12 q / 2 kv heads, bias), narrow and shallow for the CPU suite
        return pb.ModelSpec("pin-qwen2", 2, 1536, 12, 2, 128, 1024, 2048, qkv_bias=True, rope_theta=1e6)
    if kind == "qwen3":  # C3 head layout (32 q / 8 kv heads, q/k-norm, no bias)
        return pb.ModelSpec("pin-qwen3", 2, 512, 32, 8, 128, 768, 2048, qk_norm=True, rope_theta=1e6)
    # C5 head layout (28 q / 4 kv heads, bias, untied lm_head, theta 1e4)
    return pb.ModelSpec("pin-r1", 2, 896, 28, 4, 128, 640, 2048, qkv_bias=True, tied_embeddings=False,
                        rope_theta=1e4)


def _weights(spec):
    w = random_weights(spec, seed=3, std=0.05)
    g = torch.Generator().manual_seed(9)
    for k in list(w):
        if "norm" in k:
            w[k] = (1.0 + 0.2 * torch.randn(w[k].shape, generator=g)).to(torch.bfloat16)
        if k.endswith("bqkv"):
            w[k] = (0.2 * torch.randn(w[k].shape, generator=g)).to(torch.bfloat16)
    return w


def _hf_model(spec, w):
    common = dict(vocab_size=spec.vocab, hidden_size=spec.d_model, intermediate_size=spec.d_ff,
                  num_hidden_layers=spec.n_layers, num_attention_heads=spec.n_q_heads,
                  num_key_value_heads=spec.n_kv_heads, head_dim=spec.head_dim, rms_norm_eps=spec.norm_eps,
                  tie_word_embeddings=spec.tied_embeddings, max_position_embeddings=4096,
                  rope_parameters={"rope_type": "default", "rope_theta": spec.rope_theta})
    if spec.qk_norm:
        cfg = transformers.Qwen3Config(attention_bias=False, **common)
        model = transformers.Qwen3ForCausalLM(cfg)
    else:
        cfg = transformers.Qwen2Config(**common)
        model = transformers.Qwen2ForCausalLM(cfg)
    model = model.float().eval()
    hq, hk, hd = spec.n_q_heads, spec.n_kv_heads, spec.head_dim
    sd = {"model.embed_tokens.weight": w["embed"], "model.norm.weight": w["final_norm"].view(-1)}
    sd["lm_head.weight"] = w["lm_head"] if not spec.tied_embeddings else w["embed"]
    for l in range(spec.n_layers):
        p, q = f"layers.{l}.", f"model.layers.{l}."
        qkv = w[p + "wqkv"]
        sd[q + "self_attn.q_proj.weight"] = qkv[: hq * hd]
        sd[q + "self_attn.k_proj.weight"] = qkv[hq * hd: (hq + hk) * hd]
        sd[q + "self_attn.v_proj.weight"] = qkv[(hq + hk) * hd:]
        if spec.qkv_bias:
            b = w[p + "bqkv"].view(-1)
            sd[q + "self_attn.q_proj.bias"] = b[: hq * hd]
            sd[q + "self_attn.k_proj.bias"] = b[hq * hd: (hq + hk) * hd]
            sd[q + "self_attn.v_proj.bias"] = b[(hq + hk) * hd:]
        if spec.qk_norm:
            sd[q + "self_attn.q_norm.weight"] = w[p + "q_norm"].view(-1)
            sd[q + "self_attn.k_norm.weight"] = w[p + "k_norm"].view(-1)
        sd[q + "self_attn.o_proj.weight"] = w[p + "wo"]
        gate, up = split_gate_up(w[p + "wgu"])
        sd[q + "mlp.gate_proj.weight"] = gate
        sd[q + "mlp.up_proj.weight"] = up
        sd[q + "mlp.down_proj.weight"] = w[p + "wd"]
        sd[q + "input_layernorm.weight"] = w[p + "attn_norm"].view(-1)
        sd[q + "post_attention_layernorm.weight"] = w[p + "mlp_norm"].view(-1)
    missing, unexpected = model.load_state_dict({k: v.float() for k, v in sd.items()}, strict=False)
    assert not unexpected, unexpected
    assert all("rotary" in k for k in missing), missing
    return model


@pytest.mark.parametrize("kind", ["qwen2", "qwen3", "r1"])
def test_cpu_oracle_matches_transformers(kind):
    spec = _spec(kind)
    w = _weights(spec)
    model = _hf_model(spec, w)
    dec = CpuDecoder(spec, w, round_bf16=False)
    toks = [int(t) for t in pb.synthetic_prompt(1, 0, 37, spec.vocab)]
    with torch.no_grad():
        ref = model(torch.tensor([toks])).logits[0].double()
        mine = dec.forward(toks, dec.new_cache(), 0, want_logits="all").double()
    assert mine.shape == ref.shape
    err = (mine - ref).abs().max().item()
    assert err <= TOL, f"max |delta logit| {err:.2e} (logit scale {ref.abs().max().item():.2f})"
    # incremental decode through the oracle's KV cache (the path score() uses) agrees as well
    cache = dec.new_cache()
    dec.forward(toks[:-5], cache, 0, want_logits=False)
    for j in range(5):
        pos = len(toks) - 5 + j
        z = dec.forward([toks[pos]], cache, pos).double()
        assert (z - ref[pos]).abs().max().item() <= TOL
