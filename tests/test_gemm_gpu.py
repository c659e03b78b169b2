"""Tensor-core 3xTF32 GEMM (qpinn_gemm_f32, tc_gemm.cu) against float64.

C = A B^T must be FP32-class: max |C - C_f64| <= 3e-6 max |C_f64| (cuBLAS
SIMT fp32 lands at ~7e-7 on the same inputs at K = 256; the split-operand
tensor-core path at ~3.5e-7).  Ragged M, N < 16, N > 128 (several N tiles)
and K not a multiple of the 32-wide pipeline stage are covered."""
import pytest
import torch

from paper_2506_23246_b200 import _native as N

pytestmark = pytest.mark.gpu


def _gemm(A, B):
    lib = N.lib()
    M, K = A.shape
    n = B.shape[0]
    C = torch.full((M, n), float("nan"), dtype=torch.float32, device="cuda")
    ws = torch.empty(lib.qpinn_gemm_f32_workspace_bytes(n, K), dtype=torch.uint8, device="cuda")
    N.check(lib.qpinn_gemm_f32(M, n, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
                               C.data_ptr(), C.stride(0), ws.data_ptr(), ws.numel(),
                               N.stream_ptr()), "qpinn_gemm_f32")
    return C


@pytest.mark.parametrize("M,n,K", [(128, 128, 32), (1000, 128, 256), (300, 256, 128),
                                   (513, 7, 128), (4096, 64, 96), (77, 200, 40), (1, 16, 4),
                                   (70000, 128, 256)])
def test_gemm_f32_matches_f64(M, n, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + n * 3 + K)
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(n, K, device="cuda", generator=g) / K ** 0.5
    C = _gemm(A, B)
    ref = A.double() @ B.double().T
    assert torch.isfinite(C).all()
    err = (C.double() - ref).abs().max().item()
    assert err <= 3e-6 * ref.abs().max().item(), err


def test_gemm_f32_deterministic():
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(20000, 256, device="cuda", generator=g)
    B = torch.randn(128, 256, device="cuda", generator=g)
    assert torch.equal(_gemm(A, B), _gemm(A, B))


def test_gemm_rejects_unaligned_rows():
    A = torch.randn(64, 10, device="cuda")
    B = torch.randn(16, 10, device="cuda")
    with pytest.raises(Exception):
        _gemm(A, B)


def _gemm_atb(X, G):
    lib = N.lib()
    rows, m = X.shape
    n = G.shape[1]
    C = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
    ws = torch.empty(max(1, lib.qpinn_gemm_f32_atb_workspace_bytes(rows, m, n)), dtype=torch.uint8,
                     device="cuda")
    N.check(lib.qpinn_gemm_f32_atb(rows, m, n, X.data_ptr(), X.stride(0), G.data_ptr(), G.stride(0),
                                   C.data_ptr(), ws.data_ptr(), ws.numel(), N.stream_ptr()),
            "qpinn_gemm_f32_atb")
    return C


@pytest.mark.parametrize("rows,m,n", [(32, 128, 128), (1000, 128, 128), (4097, 256, 128),
                                      (300, 7, 128), (262144, 256, 128), (70001, 128, 36),
                                      (262144, 128, 7)])
def test_gemm_f32_atb_matches_f64(rows, m, n):
    """The weight-gradient kernel (X^T G, reduction over rows; A = X^T split into
    TMEM, B = G split in shared memory) against float64, ragged rows and columns."""
    g = torch.Generator(device="cuda").manual_seed(rows + 5 * m + n)
    pad = lambda k: (k + 3) // 4 * 4  # noqa: E731  (row strides are multiples of 4)
    X = torch.randn(rows, pad(m), device="cuda", generator=g)[:, :m]
    G = (torch.randn(rows, pad(n), device="cuda", generator=g) / rows ** 0.5)[:, :n]
    C = _gemm_atb(X, G)
    ref = X.double().T @ G.double()
    assert torch.isfinite(C).all()
    err = (C.double() - ref).abs().max().item()
    assert err <= 3e-6 * ref.abs().max().item(), err
    assert torch.equal(C, _gemm_atb(X, G))  # fixed-order chunk sum


def test_gemm_f32_repeatable_under_load():
    """Bitwise repeatability over many launches at the step's shapes: guards the
    raw A stage's hand-back to TMA (generic-proxy reads, then an async-proxy
    refill; without the proxy fence about 1 launch in 50 had a row computed from
    the next k-block's data, scripts/race_gemm.py)."""
    for (M, n, K) in [(65536, 256, 128), (262144, 128, 128)]:
        g = torch.Generator(device="cuda").manual_seed(M + n)
        A = torch.randn(M, K, device="cuda", generator=g)
        B = torch.randn(n, K, device="cuda", generator=g) / K ** 0.5
        ref = _gemm(A, B)
        for _ in range(120):
            assert torch.equal(_gemm(A, B), ref)
