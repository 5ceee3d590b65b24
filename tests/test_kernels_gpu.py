"""Kernel numerics against plain PyTorch fp32 references of the same op."""

import ctypes as C

import pytest

torch = pytest.importorskip("torch")

from paper_2509_18521_b200 import _capi  # noqa: E402

pytestmark = pytest.mark.gpu


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


@pytest.mark.parametrize("bn", [32, 64, 128, 256, -128, -256])  # < 0: no-swap schedule, -bn weight rows per tile
@pytest.mark.parametrize("shape", [(256, 128, 1), (512, 1536, 37), (2048, 1536, 300), (384, 256, 1000)])
@pytest.mark.parametrize("epi", [0, 1, 2, 16, 17, 18])  # +16: deterministic split-K enabled
def test_tcgen05_gemm_matches_torch(bn, shape, epi):
    N, K, M = shape
    split = epi >= 16
    epi_code, epi = epi, epi & 15
    g = torch.Generator(device="cuda").manual_seed(N * 7 + K + M)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    A = (torch.randn(M, K, device="cuda", generator=g)).to(torch.bfloat16)
    bias = (torch.randn(N, device="cuda", generator=g) * 0.1).to(torch.bfloat16) if epi == 0 else None
    ref = A.float() @ W.float().t()
    if epi == 0:
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ref = ref + bias.float()
    elif epi == 1:
        out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    else:
        base = torch.randn(M, N, device="cuda", generator=g)
        out = base.clone()
        ref = ref + base
    if bn < 0:
        bn, epi_code = -bn, epi_code + 64
    _capi.call("ab_debug_gemm", _ptr(W), _ptr(A), _ptr(out), _ptr(bias), N, K, M, bn, epi_code)
    torch.cuda.synchronize()
    if split:  # deterministic: a second run is bit-identical
        again = out.clone() if epi != 2 else base.clone()
        _capi.call("ab_debug_gemm", _ptr(W), _ptr(A), _ptr(again), _ptr(bias), N, K, M, bn, epi_code)
        torch.cuda.synchronize()
        assert torch.equal(again, out)
    tol = 2e-2 if epi == 0 else 2e-3
    torch.testing.assert_close(out.float(), ref, rtol=tol, atol=tol * max(1.0, ref.abs().max().item() * 0.01))


@pytest.mark.parametrize("epi", [3, 19, 3 + 64, 19 + 64])  # +64: activation rows on the UMMA M side
def test_tcgen05_gemm_swiglu_epilogue(epi):
    N, K, M = 512, 1024, 77  # N = 2 * features, rows interleaved in 64-row halves per 128-row tile
    g = torch.Generator(device="cuda").manual_seed(5)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
    _capi.call("ab_debug_gemm", _ptr(W), _ptr(A), _ptr(out), None, N, K, M, 256 if epi & 64 else 64, epi)
    acc = A.float() @ W.float().t()
    t = acc.view(M, N // 128, 2, 64)
    ref = (torch.nn.functional.silu(t[:, :, 0]) * t[:, :, 1]).reshape(M, N // 2)
    torch.testing.assert_close(out.float(), ref, rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("rows", [1, 17, 64, 200, 333, 1024])
@pytest.mark.parametrize("shape_epi", [((1536, 1536), 2), ((2048, 1536), 0), ((512, 1024), 3), ((1536, 8960), 2),
                                       ((384, 640), 1)])
@pytest.mark.parametrize("split", [0, 16, 256])  # 16: cluster split-K plan, 256: CTA-pair plan
def test_tcgen05_gemm_auto_schedule(rows, shape_epi, split):
    """The decode configuration: tile width and split-K picked on the device from the row count."""
    (N, K), epi = shape_epi
    M = rows
    g = torch.Generator(device="cuda").manual_seed(N + K + M)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    acc = A.float() @ W.float().t()
    bias = None
    if epi == 3:
        out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
        t = acc.view(M, N // 128, 2, 64)
        ref = (torch.nn.functional.silu(t[:, :, 0]) * t[:, :, 1]).reshape(M, N // 2)
    elif epi == 0:
        bias = (torch.randn(N, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ref = acc + bias.float()
    elif epi == 1:
        out = torch.empty(M, N, device="cuda", dtype=torch.float32)
        ref = acc
    else:
        base = torch.randn(M, N, device="cuda", generator=g)
        out = base.clone()
        ref = acc + base
    _capi.call("ab_debug_gemm", _ptr(W), _ptr(A), _ptr(out), _ptr(bias), N, K, M, 256, epi + split + 32)
    torch.cuda.synchronize()
    tol = 2e-2 if epi in (0, 3) else 2e-3
    torch.testing.assert_close(out.float(), ref, rtol=tol, atol=tol * max(1.0, ref.abs().max().item() * 0.01))


@pytest.mark.parametrize("shape", [(256, 128, 1), (512, 1536, 37), (2048, 1536, 300), (384, 256, 1000),
                                   (1536, 8960, 600)])
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
def test_tcgen05_gemm_cta_pair(shape, epi):
    """The CTA-pair schedule (cta_group::2, 256 x 256 tile split over two SMs), forced."""
    N, K, M = shape
    if epi == 3 and N % 256:
        pytest.skip("SwiGLU pair tiles need N % 256 == 0")
    g = torch.Generator(device="cuda").manual_seed(N + 3 * K + M)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    acc = A.float() @ W.float().t()
    bias = None
    if epi == 3:
        out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
        t = acc.view(M, N // 128, 2, 64)
        ref = (torch.nn.functional.silu(t[:, :, 0]) * t[:, :, 1]).reshape(M, N // 2)
    elif epi == 0:
        bias = (torch.randn(N, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ref = acc + bias.float()
    elif epi == 1:
        out = torch.empty(M, N, device="cuda", dtype=torch.float32)
        ref = acc
    else:
        base = torch.randn(M, N, device="cuda", generator=g)
        out = base.clone()
        ref = acc + base
    # bit 8: cluster of 2 (a pair plan), bit 7: fixed schedule code; 0x4000 = CTA pair
    _capi.call("ab_debug_gemm", _ptr(W), _ptr(A), _ptr(out), _ptr(bias), N, K, M, 0x4000, epi + 256 + 128)
    torch.cuda.synchronize()
    tol = 2e-2 if epi in (0, 3) else 2e-3
    torch.testing.assert_close(out.float(), ref, rtol=tol, atol=tol * max(1.0, ref.abs().max().item() * 0.01))


@pytest.mark.parametrize("shape", [(1536, 1536, 384), (1536, 8960, 256), (384, 640, 1000), (1536, 8960, 37)])
@pytest.mark.parametrize("code", [1 | (6 << 1) | (2 << 5), 0 | (7 << 1) | (4 << 5), 1 | (5 << 1) | (8 << 5)])
def test_tcgen05_gemm_reduce_add_split(shape, code):
    """fp32 residual GEMM with split-K partials reduce-added by TMA (no cluster); fixed schedules."""
    N, K, M = shape
    if _capi.lib().ab_debug_gemm_sched(N, K, M, 256, 1, 148, 0x40000000 | 0x8000 | code, 2) == 0:
        pytest.skip("schedule not valid for this shape (too few k-blocks per split)")
    g = torch.Generator(device="cuda").manual_seed(N + K + M + code)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    base = torch.randn(M, N, device="cuda", generator=g)
    out = base.clone()
    # bit 10: cluster-of-1 plan allowing reduce-add split-K, bit 7: fixed code, 0x8000: reduce-add split
    _capi.call("ab_debug_gemm", _ptr(W), _ptr(A), _ptr(out), None, N, K, M, 0x8000 | code, 2 + 1024 + 128)
    torch.cuda.synchronize()
    ref = base + A.float() @ W.float().t()
    torch.testing.assert_close(out, ref, rtol=2e-3, atol=2e-3 * max(1.0, ref.abs().max().item() * 0.01))


@pytest.mark.parametrize("shape", [(19456, 2560, 64), (6144, 2560, 64), (1536, 1536, 384), (2560, 9728, 100),
                                   (384, 640, 1000)])
@pytest.mark.parametrize("code", [0x10000 | 1 | (6 << 1) | (1 << 5), 0x10000 | 1 | (7 << 1) | (1 << 5),
                                  0x10000 | 0 | (7 << 1) | (1 << 5), 1 | (6 << 1) | (3 << 5), 1 | (7 << 1) | (7 << 5)])
def test_tcgen05_gemm_stream_k_and_odd_splits(shape, code):
    """Stream-K reduce-add ranges (0x10000: every CTA streams an equal contiguous range of (tile,
    k-block pair) work, split over tile boundaries) and non-power-of-two reduce-add split counts."""
    N, K, M = shape
    if _capi.lib().ab_debug_gemm_sched(N, K, M, 256, 1, 148, 0x40000000 | 0x8000 | code, 2) == 0:
        pytest.skip("schedule not valid for this shape")
    g = torch.Generator(device="cuda").manual_seed(N + K + M + code)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    base = torch.randn(M, N, device="cuda", generator=g)
    out = base.clone()
    _capi.call("ab_debug_gemm", _ptr(W), _ptr(A), _ptr(out), None, N, K, M, 0x8000 | code, 2 + 1024 + 128)
    torch.cuda.synchronize()
    ref = base + A.float() @ W.float().t()
    torch.testing.assert_close(out, ref, rtol=2e-3, atol=2e-3 * max(1.0, ref.abs().max().item() * 0.01))
