"""torch-CPU fp32 reference decoder — TEST INFRASTRUCTURE ONLY.

The reference has no transformer (its engine is the d0 + d1*b cost model,
src/april_sim/engine.py:167-171), so decode numerics are pinned
by this restatement of the B200 engine's documented math:

  x (fp32 residual) = bf16 embedding row
  per layer:  xn  = bf16(x * rsqrt(mean(x^2) + eps) * w_attn_norm)
              qkv = bf16(xn @ Wqkv^T + b)            (fp32 accumulate)
              q,k = [qk-norm: bf16(rmsnorm_head(.) * w)] -> RoPE(rotate-half, fp32) -> bf16
              att = softmax(q k^T / sqrt(hd)) v       (fp32; causal over the sequence)
              x  += bf16(att) @ Wo^T
              xn  = bf16(rmsnorm(x) * w_mlp_norm)
              h   = bf16(silu(xn @ Wg^T) * (xn @ Wu^T))
              x  += h @ Wd^T
  logits = bf16(rmsnorm(x) * w_final) @ E^T           (fp32)
  greedy token = argmax (lowest index on ties); logp = log_softmax(logits / T)[tok]

Weights are read back from the engine (`Engine.export_weights()`), so the
oracle and the GPU run on identical bf16 parameters.  The gate/up matrix is
stored tile-interleaved on the device (per 128-row tile: 64 gate rows, then
the 64 matching up rows); `split_gate_up` undoes that.
"""

from __future__ import annotations

import math

import torch


def split_gate_up(wgu: torch.Tensor):
    two_f, d = wgu.shape
    t = wgu.view(two_f // 128, 2, 64, d)
    return t[:, 0].reshape(two_f // 2, d), t[:, 1].reshape(two_f // 2, d)


def _bf(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).float()


def random_weights(spec, seed: int = 0, std: float = 0.02) -> dict:
    """CPU-generated weights of the engine's layout (for CPU-only baselines)."""
    g = torch.Generator().manual_seed(seed)
    d, f, hq, hk, hd, V = spec.d_model, spec.d_ff, spec.n_q_heads, spec.n_kv_heads, spec.head_dim, spec.vocab
    qkv = (hq + 2 * hk) * hd

    def rnd(r, c):
        return (torch.randn(r, c, generator=g) * std).to(torch.bfloat16)

    w = {"embed": rnd(V, d), "final_norm": torch.ones(1, d, dtype=torch.bfloat16)}
    if not spec.tied_embeddings:
        w["lm_head"] = rnd(V, d)
    for l in range(spec.n_layers):
        p = f"layers.{l}."
        w[p + "attn_norm"] = torch.ones(1, d, dtype=torch.bfloat16)
        w[p + "wqkv"] = rnd(qkv, d)
        if spec.qkv_bias:
            w[p + "bqkv"] = rnd(1, qkv)
        if spec.qk_norm:
            w[p + "q_norm"] = torch.ones(1, hd, dtype=torch.bfloat16)
            w[p + "k_norm"] = torch.ones(1, hd, dtype=torch.bfloat16)
        w[p + "wo"] = rnd(d, hq * hd)
        w[p + "mlp_norm"] = torch.ones(1, d, dtype=torch.bfloat16)
        w[p + "wgu"] = rnd(2 * f, d)
        w[p + "wd"] = rnd(d, f)
    return w


class CpuDecoder:
    """round_bf16=False drops the engine's bf16 activation roundings (pure fp32 math on the bf16
    weights): the form `tests/test_cpu_model_pin.py` checks against transformers' Qwen2 / Qwen3.
    compute_dtype=torch.float64 keeps the roundings but sums in fp64: the distance between the fp32
    and fp64 forms is the noise floor of the rounding scheme itself (tools/noise_floor.py)."""

    def __init__(self, spec, weights: dict, threads: int | None = None, round_bf16: bool = True,
                 compute_dtype=torch.float32):
        if threads:
            torch.set_num_threads(threads)
        self.s = spec
        dt = self.dt = compute_dtype  # float64: the same roundings with exact-ish sums (noise-floor runs)
        self._bf = (lambda x: x.to(torch.bfloat16).to(dt)) if round_bf16 else (lambda x: x)
        w = {k: v.to(dt) for k, v in weights.items()}
        self.embed = w["embed"]
        self.lm_head = w.get("lm_head", self.embed)
        self.final_norm = w["final_norm"].view(-1)
        self.layers = []
        for l in range(spec.n_layers):
            p = f"layers.{l}."
            g, u = split_gate_up(w[p + "wgu"])
            self.layers.append(dict(
                attn_norm=w[p + "attn_norm"].view(-1), wqkv=w[p + "wqkv"],
                bqkv=w[p + "bqkv"].view(-1) if p + "bqkv" in w else None,
                q_norm=w[p + "q_norm"].view(-1) if p + "q_norm" in w else None,
                k_norm=w[p + "k_norm"].view(-1) if p + "k_norm" in w else None,
                wo=w[p + "wo"], mlp_norm=w[p + "mlp_norm"].view(-1), wg=g, wu=u, wd=w[p + "wd"]))
        hd = spec.head_dim
        inv = 1.0 / torch.pow(torch.tensor(spec.rope_theta, dtype=torch.float32),
                              torch.arange(0, hd, 2, dtype=torch.float32) / hd)
        self.inv_freq = inv

    def _rms(self, x, w):
        return self._bf(x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + self.s.norm_eps) * w)

    def _rope(self, x, pos):  # x [T, H, hd] fp32, pos [T]
        ang = pos.float()[:, None] * self.inv_freq[None, :]
        c, s = torch.cos(ang)[:, None, :].to(self.dt), torch.sin(ang)[:, None, :].to(self.dt)
        h = x.shape[-1] // 2
        a, b = x[..., :h], x[..., h:]
        return torch.cat([a * c - b * s, b * c + a * s], dim=-1)

    def new_cache(self):
        return [dict(k=[], v=[]) for _ in range(self.s.n_layers)]

    @torch.no_grad()
    def forward(self, tokens: list[int], cache, start_pos: int, want_logits: bool = True):
        """Run `tokens` at positions start_pos.. (causal over cache + tokens)."""
        s = self.s
        T = len(tokens)
        hq, hk, hd = s.n_q_heads, s.n_kv_heads, s.head_dim
        pos = torch.arange(start_pos, start_pos + T)
        x = self.embed[torch.tensor(tokens)].clone()
        for l, L in enumerate(self.layers):
            xn = self._rms(x, L["attn_norm"])
            qkv = xn @ L["wqkv"].t()
            if L["bqkv"] is not None:
                qkv = qkv + L["bqkv"]
            qkv = self._bf(qkv)
            q = qkv[:, : hq * hd].view(T, hq, hd)
            k = qkv[:, hq * hd: (hq + hk) * hd].view(T, hk, hd)
            v = qkv[:, (hq + hk) * hd:].view(T, hk, hd)
            if L["q_norm"] is not None:
                q = self._rms(q, L["q_norm"])
                k = self._rms(k, L["k_norm"])
            q = self._bf(self._rope(q, pos))
            k = self._bf(self._rope(k, pos))
            cache[l]["k"].append(k)
            cache[l]["v"].append(v)
            K = torch.cat(cache[l]["k"], 0)
            V = torch.cat(cache[l]["v"], 0)
            n = K.shape[0]
            g = hq // hk
            Kx = K.repeat_interleave(g, dim=1)  # [n, hq, hd]
            Vx = V.repeat_interleave(g, dim=1)
            sc = torch.einsum("thd,nhd->htn", q, Kx) / math.sqrt(hd)
            mask = torch.arange(n)[None, :] > (start_pos + torch.arange(T))[:, None]
            sc = sc.masked_fill(mask[None], float("-inf"))
            p = torch.softmax(sc, dim=-1)
            att = self._bf(torch.einsum("htn,nhd->thd", p, Vx).reshape(T, hq * hd))
            x = x + att @ L["wo"].t()
            xn = self._rms(x, L["mlp_norm"])
            h = self._bf(torch.nn.functional.silu(xn @ L["wg"].t()) * (xn @ L["wu"].t()))
            x = x + h @ L["wd"].t()
        if not want_logits:
            return None
        if want_logits == "all":
            return self._rms(x, self.final_norm) @ self.lm_head.t()
        xn = self._rms(x[-1:], self.final_norm)
        return (xn @ self.lm_head.t())[0]

    @torch.no_grad()
    def decode_batch_rate(self, batch: int, ctx: int, iters: int, seed: int = 0) -> dict:
        """CPU baseline: `iters` decode iterations of `batch` sequences whose caches hold
        `ctx` tokens, same math as forward(); returns generated tokens/s."""
        import time

        s = self.s
        hq, hk, hd = s.n_q_heads, s.n_kv_heads, s.head_dim
        g = torch.Generator().manual_seed(seed)
        caches = [[torch.randn(batch, ctx + iters, hk, hd, generator=g) * 0.5 for _ in range(2)]
                  for _ in range(s.n_layers)]
        toks = torch.randint(0, s.vocab - 1, (batch,), generator=g)
        t0 = time.perf_counter()
        for it in range(iters):
            n = ctx + it + 1
            pos = torch.full((batch,), ctx + it)
            x = self.embed[toks].clone()
            for l, L in enumerate(self.layers):
                xn = self._rms(x, L["attn_norm"])
                qkv = xn @ L["wqkv"].t()
                if L["bqkv"] is not None:
                    qkv = qkv + L["bqkv"]
                qkv = self._bf(qkv)
                q = qkv[:, : hq * hd].view(batch, hq, hd)
                k = qkv[:, hq * hd: (hq + hk) * hd].view(batch, hk, hd)
                v = qkv[:, (hq + hk) * hd:].view(batch, hk, hd)
                if L["q_norm"] is not None:
                    q = self._rms(q, L["q_norm"])
                    k = self._rms(k, L["k_norm"])
                q = self._bf(self._rope(q, pos))
                K, V = caches[l]
                K[:, n - 1] = self._bf(self._rope(k, pos))
                V[:, n - 1] = v
                qg = q.view(batch, hk, hq // hk, hd)
                sc = torch.einsum("bgqd,bngd->bgqn", qg, K[:, :n]) / math.sqrt(hd)
                att = torch.einsum("bgqn,bngd->bgqd", torch.softmax(sc, -1), V[:, :n])
                x = x + self._bf(att.reshape(batch, hq * hd)) @ L["wo"].t()
                xn = self._rms(x, L["mlp_norm"])
                h = self._bf(torch.nn.functional.silu(xn @ L["wg"].t()) * (xn @ L["wu"].t()))
                x = x + h @ L["wd"].t()
            z = self._rms(x, self.final_norm) @ self.lm_head.t()
            toks = torch.argmax(z, -1)
        dt = time.perf_counter() - t0
        return {"tokens": batch * iters, "seconds": dt, "tokens_per_s": batch * iters / dt,
                "threads": torch.get_num_threads()}

    @torch.no_grad()
    def score_all(self, prompt: list[int], generated: list[int], temperature: float = 1.0):
        """Teacher-forced scoring of a whole generated sequence in ONE causal pass (same math as
        forward() token by token, but matrix-matrix; used for the full-depth greedy tests).
        Returns numpy arrays per generated position: oracle argmax, margin z[argmax] - z[token],
        log_softmax(z / T)[token], top-2 margin."""
        seq = list(prompt) + list(generated[:-1])
        z = self.forward(seq, self.new_cache(), 0, want_logits="all")[len(prompt) - 1:]
        tok = torch.tensor(list(generated), dtype=torch.long)
        am = torch.argmax(z, -1)
        zt = z.gather(1, tok[:, None])[:, 0]
        margin = z.gather(1, am[:, None])[:, 0] - zt
        lp = torch.log_softmax(z.double() / temperature, dim=-1).gather(1, tok[:, None])[:, 0]
        top2 = torch.topk(z, 2, dim=-1).values
        return dict(argmax=am.numpy(), margin=margin.numpy(), logp=lp.numpy(),
                    top2=(top2[:, 0] - top2[:, 1]).numpy())

    @torch.no_grad()
    def score(self, prompt: list[int], generated: list[int], temperature: float = 1.0):
        """Teacher-forced pass: per generated position, (oracle argmax, its margin over the
        GPU token, oracle logprob of the GPU token, top-2 margin)."""
        cache = self.new_cache()
        self.forward(prompt[:-1], cache, 0, want_logits=False)
        out = []
        tok = prompt[-1]
        pos = len(prompt) - 1
        for g in generated:
            z = self.forward([tok], cache, pos)
            top2 = torch.topk(z, 2)
            am = int(torch.argmax(z))
            lp = torch.log_softmax(z.double() / temperature, dim=-1)
            out.append(dict(argmax=am, margin=float(z[am] - z[g]), logp=float(lp[g]),
                            top2=float(top2.values[0] - top2.values[1])))
            tok = g
            pos += 1
        return out
