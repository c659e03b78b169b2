"""Role wait-time breakdown of the tcgen05 GEMM (exp/prof.so built with -DQPINN_GEMM_PROF):
cycles CTA 0's roles spent blocked on each mbarrier, relative to the kernel time."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_23246_b200 import _native as N  # noqa: E402

lib = N.lib()
prof = lib.qpinn_gemm_prof
prof.argtypes = [C.c_void_p]
names = ["A prod wait raw_empty", "B prod wait b_empty", "MMA wait tempty", "MMA wait conv",
         "MMA wait b_full", "conv(w0) wait op_empty", "conv(w0) wait raw_full",
         "epi(w4) wait tfull", "epi(w4) store phase", "kernel (CTA0 thread0)"]
for (M, n, K) in [(262144, 256, 256), (262144, 128, 256), (262144, 128, 128)]:
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(n, K, device="cuda")
    Cm = torch.empty((M, n), device="cuda")
    ws = torch.empty(lib.qpinn_gemm_f32_workspace_bytes(n, K), dtype=torch.uint8, device="cuda")
    def go():
        N.check(lib.qpinn_gemm_f32(M, n, K, A.data_ptr(), K, B.data_ptr(), K, Cm.data_ptr(), n,
                                   ws.data_ptr(), ws.numel(), N.stream_ptr()), "gemm")
    go()
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 16)()
    prof(buf)
    for _ in range(10):
        go()
    torch.cuda.synchronize()
    prof(buf)
    tot = buf[9]
    print(f"M={M} N={n} K={K}: kernel {tot / 10:.0f} cycles/launch")
    for i, nm in enumerate(names[:9]):
        print(f"   {nm:26s} {buf[i] / tot * 100:6.1f} %")
