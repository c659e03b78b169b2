"""Tensor-core 3xTF32 GEMM (qpinn_gemm_f32): accuracy vs float64 and timing."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_23246_b200 import _native as N  # noqa: E402


def gemm(A, B, C_=None):
    lib = N.lib()
    M, K = A.shape
    n = B.shape[0]
    C_ = torch.empty((M, n), dtype=torch.float32, device="cuda") if C_ is None else C_
    ws = torch.empty(lib.qpinn_gemm_f32_workspace_bytes(n, K), dtype=torch.uint8, device="cuda")
    N.check(lib.qpinn_gemm_f32(M, n, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
                               C_.data_ptr(), C_.stride(0), ws.data_ptr(), ws.numel(),
                               N.stream_ptr()), "gemm")
    return C_


torch.manual_seed(0)
for (M, n, K) in [(128, 128, 32), (1000, 128, 256), (300, 256, 128), (513, 7, 128), (4096, 64, 96),
                  (262144, 128, 256), (262144, 128, 128), (262144, 256, 128), (262144, 256, 256)]:
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(n, K, device="cuda") / K ** 0.5
    Cg = gemm(A, B)
    torch.cuda.synchronize()
    ref = A.double() @ B.double().T
    err = (Cg.double() - ref).abs().max().item()
    scale = ref.abs().max().item()
    f32 = (A @ B.T).double()
    err32 = (f32 - ref).abs().max().item()
    line = f"M={M} N={n} K={K}: max|err| {err:.3e} (rel {err / scale:.2e}); torch fp32 {err32:.3e}"
    if M >= 65536:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            gemm(A, B, Cg)
        e0.record()
        for _ in range(20):
            gemm(A, B, Cg)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        fl = 2 * M * n * K
        by = 4 * (M * K + M * n)
        line += f" | {ms * 1e3:.1f} us  {fl / ms / 1e9:.1f} TFLOP/s (x3 MMA)  {by / ms / 1e6:.0f} GB/s"
        e0.record()
        for _ in range(20):
            torch.mm(A, B.T, out=Cg)
        e1.record()
        torch.cuda.synchronize()
        line += f" | torch fp32 {e0.elapsed_time(e1) / 20 * 1e3:.1f} us"
    print(line, flush=True)


def atb(X, G):
    lib = N.lib()
    rows, m = X.shape
    n = G.shape[1]
    C_ = torch.empty((m, n), dtype=torch.float32, device="cuda")
    ws = torch.empty(lib.qpinn_gemm_f32_atb_workspace_bytes(rows, m, n), dtype=torch.uint8,
                     device="cuda")
    N.check(lib.qpinn_gemm_f32_atb(rows, m, n, X.data_ptr(), X.stride(0), G.data_ptr(), G.stride(0),
                                   C_.data_ptr(), ws.data_ptr(), ws.numel(), N.stream_ptr()), "atb")
    return C_


for (rows, m, n) in [(64, 128, 128), (1000, 96, 40), (262144, 256, 128), (262144, 128, 128), (262144, 256, 256),
                     (70001, 132, 200)]:
    X = torch.randn(rows, m, device="cuda")
    G = torch.randn(rows, n, device="cuda")
    Cg = atb(X, G)
    torch.cuda.synchronize()
    ref = X.double().T @ G.double()
    err = (Cg.double() - ref).abs().max().item()
    f32 = (X.T @ G).double()
    line = (f"atb rows={rows} m={m} n={n}: max|err| {err:.3e} (rel {err / ref.abs().max().item():.2e});"
            f" torch fp32 {(f32 - ref).abs().max().item():.3e}")
    if rows >= 262144:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            atb(X, G)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        e0.record()
        for _ in range(10):
            torch.mm(X.T, G)
        e1.record()
        torch.cuda.synchronize()
        line += f" | {ms * 1e3:.1f} us vs torch fp32 {e0.elapsed_time(e1) / 10 * 1e3:.1f} us"
    print(line, flush=True)
