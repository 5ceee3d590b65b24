"""K3 (paged GQA decode attention) against a torch fp32 reference, kernel level.

`ab_debug_decode_attn` runs exactly the engine's `k_decode_attn` launch over a caller-built
single-layer paged pool: random bf16 K/V pages scattered over the pool (a random page permutation,
so no row's pages are contiguous), random bf16 q, per-row context lengths.  The reference is
softmax(q k^T / sqrt(hd)) v in fp32 over the same bf16 K/V, with the GQA head mapping
q head h -> kv head h // (hq / hk).

Tolerance (stated, elementwise): |out - ref| <= ATOL + RTOL * (P |V|) with ATOL = 2e-3, RTOL = 2e-2,
where P |V| = softmax(q k^T / sqrt(hd)) |v| is the magnitude of the terms being summed (the forward
error bound of a weighted sum: when positive and negative values cancel, ref is small but each
term's rounding error is not).  The kernel rounds the probabilities to bf16 for P.V
(flash-attention-2 register layout) and its output to bf16 (2^-9 relative each); the fp32
reference does neither.

Cases cover the configs the bench runs and their edges: rows b in {1, 7, 64, 1024}; contexts
{1, 63, 65, 100, 300, 1400, 4096, 16640}; (hq, hk) in {(12, 2) C2, (32, 8) C3/C4, (28, 4) C5};
pages of 16 and 64 tokens; the engine's own per-iteration split choice and forced multi-split
schedules, so the last-CTA split merge (split order) runs on every shape.  Every case is run twice
and must be bit-identical (the split merge is deterministic by construction).
"""

import ctypes as C
import math

import numpy as np
import pytest

from paper_2509_18521_b200 import _capi as capi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ATOL, RTOL = 2e-3, 2e-2
HEADS = {"c2": (12, 2), "c3": (32, 8), "c5": (28, 4)}


def _contexts(kind, rng):
    if kind == "single_long":
        return [16640]
    if kind == "single_short":
        return [100]
    if kind == "mixed7":
        return [1, 63, 65, 300, 1400, 4096, 16640]
    if kind == "b64":
        return list(rng.integers(1, 3001, size=64))
    if kind == "b1024":
        return list(rng.integers(1, 1401, size=1024))
    raise ValueError(kind)


def _build(ctx, hq, hk, hd, P, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    rows = len(ctx)
    npages_row = [math.ceil(c / P) for c in ctx]
    max_pages = max(npages_row)
    n_pages = sum(npages_row) + 3
    perm = torch.randperm(n_pages, generator=torch.Generator().manual_seed(seed)).tolist()
    bt = torch.zeros(rows, max_pages, dtype=torch.int32)
    k = 0
    for i, n in enumerate(npages_row):
        bt[i, :n] = torch.tensor(perm[k:k + n], dtype=torch.int32)
        k += n
    kv = torch.randn(n_pages, 2, hk, P, hd, generator=g, device="cuda").to(torch.bfloat16)
    q = torch.randn(rows, hq * hd, generator=g, device="cuda").to(torch.bfloat16)
    return q, kv, bt.cuda(), max_pages, n_pages


def _reference(q, kv, bt, ctx, hq, hk, hd, P):
    gq = hq // hk
    out = torch.empty(len(ctx), hq * hd, dtype=torch.float32, device="cuda")
    mag = torch.empty_like(out)
    for i, n in enumerate(ctx):
        pages = bt[i, : math.ceil(n / P)].long()
        K = kv[pages, 0].float().permute(1, 0, 2, 3).reshape(hk, -1, hd)[:, :n]  # [hk, n, hd]
        V = kv[pages, 1].float().permute(1, 0, 2, 3).reshape(hk, -1, hd)[:, :n]
        qi = q[i].float().view(hk, gq, hd)
        s = torch.einsum("kgd,knd->kgn", qi, K) / math.sqrt(hd)
        p = torch.softmax(s, -1)
        out[i] = torch.einsum("kgn,knd->kgd", p, V).reshape(-1)
        mag[i] = torch.einsum("kgn,knd->kgd", p, V.abs()).reshape(-1)
    return out, mag


def _run(q, kv, bt, max_pages, n_pages, ctx, hq, hk, hd, P, chunk):
    out = torch.empty_like(q)
    ctx_a = (C.c_int32 * len(ctx))(*[int(c) for c in ctx])
    used = C.c_int()
    capi.call("ab_debug_decode_attn", C.c_void_p(q.data_ptr()), C.c_void_p(kv.data_ptr()), n_pages, P, hk, hd,
              hq // hk, C.c_void_p(bt.data_ptr()), max_pages, ctx_a, len(ctx), chunk, C.c_void_p(out.data_ptr()),
              C.byref(used))
    return out, used.value


def _forced_chunk(ctx):
    """Smallest legal split (<= 64 splits per row): many splits on every long row."""
    return max(64, math.ceil(max(ctx) / 64 / 64) * 64)


@pytest.mark.parametrize("page", [16, 64])
@pytest.mark.parametrize("heads", ["c2", "c3", "c5"])
@pytest.mark.parametrize("kind", ["single_short", "single_long", "mixed7", "b64", "b1024"])
@pytest.mark.parametrize("split", ["engine", "forced"])
def test_decode_attention_matches_fp32_reference(kind, heads, page, split):
    hq, hk = HEADS[heads]
    hd = 128
    rng = np.random.default_rng(7)
    ctx = _contexts(kind, rng)
    q, kv, bt, max_pages, n_pages = _build(ctx, hq, hk, hd, page, seed=len(ctx) * 31 + hq)
    chunk = _forced_chunk(ctx) if split == "forced" else 0
    out, used = _run(q, kv, bt, max_pages, n_pages, ctx, hq, hk, hd, page, chunk)
    out2, _ = _run(q, kv, bt, max_pages, n_pages, ctx, hq, hk, hd, page, chunk)
    assert torch.equal(out, out2), "decode attention is not deterministic"
    if split == "forced":
        assert max(math.ceil(c / used) for c in ctx) > 1 or max(ctx) <= 64  # the split merge ran
    ref, mag = _reference(q, kv, bt, ctx, hq, hk, hd, page)
    err = (out.float() - ref).abs()
    bound = ATOL + RTOL * mag
    bad = (err > bound).nonzero()
    assert bad.numel() == 0, (f"{bad.shape[0]} elements out of tolerance; worst |err| {err.max().item():.3e} "
                              f"at {bad[0].tolist()} (chunk {used})")


def test_decode_attention_head_dim_64_and_gqa_8():
    """head_dim 64 (the tiny model) and the widest supported GQA group (8 q heads per kv head)."""
    for hq, hk, hd in ((4, 2, 64), (16, 2, 64), (16, 2, 128)):
        ctx = [1, 64, 129, 777, 2049]
        q, kv, bt, max_pages, n_pages = _build(ctx, hq, hk, hd, 16, seed=hq * hd)
        for chunk in (0, 64):
            out, _ = _run(q, kv, bt, max_pages, n_pages, ctx, hq, hk, hd, 16, chunk)
            ref, mag = _reference(q, kv, bt, ctx, hq, hk, hd, 16)
            assert ((out.float() - ref).abs() <= ATOL + RTOL * mag).all()


def test_decode_attention_rejects_bad_arguments():
    q, kv, bt, max_pages, n_pages = _build([100], 12, 2, 128, 64, seed=1)
    with pytest.raises(Exception):
        _run(q, kv, bt, max_pages, n_pages, [100 * 64], 12, 2, 128, 64, 0)  # context past the block table
    with pytest.raises(Exception):
        _run(q, kv, bt, max_pages, n_pages, [100], 12, 2, 128, 64, 96)  # split not a multiple of 64
