"""Bitwise repeatability of the tcgen05 GEMM (qpinn_gemm_f32) over many repeats."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_23246_b200 import _native as N  # noqa: E402

lib = N.lib()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for (M, n, K) in [(65536, 256, 128), (262144, 128, 128), (65536, 128, 256)]:
    g = torch.Generator(device="cuda").manual_seed(M + n + K)
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(n, K, device="cuda", generator=g) / K ** 0.5
    ws = torch.empty(lib.qpinn_gemm_f32_workspace_bytes(n, K), dtype=torch.uint8, device="cuda")
    ref = None
    bad = 0
    for r in range(reps):
        C = torch.full((M, n), float("nan"), device="cuda")
        N.check(lib.qpinn_gemm_f32(M, n, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
                                   C.data_ptr(), C.stride(0), ws.data_ptr(), ws.numel(),
                                   N.stream_ptr()), "gemm")
        if ref is None:
            ref = C.clone()
            continue
        if not torch.equal(C, ref):
            bad += 1
            rows = torch.nonzero((C != ref).any(1)).flatten()
            cols = torch.nonzero((C != ref).any(0)).flatten()
            print(f"M={M} N={n} K={K} rep {r}: rows {rows[:12].tolist()} ({rows.numel()}), "
                  f"cols {cols[:8].tolist()}.. ({cols.numel()}), nan {int(torch.isnan(C).sum())}", flush=True)
    print(f"M={M} N={n} K={K}: {bad}/{reps - 1} repeats differ", flush=True)
