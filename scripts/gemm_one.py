"""One tensor-core GEMM shape: a few launches (ncu captures) and event timing.
usage: gemm_one.py M N K [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_23246_b200 import _native as N  # noqa: E402

M, n, K = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (262144, 128, 256)))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
lib = N.lib()
A = torch.randn(M, K, device="cuda")
B = torch.randn(n, K, device="cuda")
C = torch.empty(M, n, device="cuda")
ws = torch.empty(lib.qpinn_gemm_f32_workspace_bytes(n, K), dtype=torch.uint8, device="cuda")


def run():
    N.check(lib.qpinn_gemm_f32(M, n, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), n,
                               ws.data_ptr(), ws.numel(), N.stream_ptr()), "gemm")


for _ in range(3):
    run()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / reps * 1e3
idx = torch.randint(0, M, (4096,), device="cuda")
ref = A[idx].double() @ B.double().T
err = ((C[idx].double() - ref).abs().max() / ref.abs().max()).item()
print(f"M={M} N={n} K={K}: {us:.1f} us, A {4 * M * K / us / 1e3:.0f} GB/s, "
      f"A+C {4 * M * (K + n) / us / 1e3:.0f} GB/s, rel err {err:.2e}")
