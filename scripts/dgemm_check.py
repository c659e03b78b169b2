import torch
M, N, K = 262144, 256, 256
a = torch.randn(M, K, device="cuda", dtype=torch.float64); b = torch.randn(K, N, device="cuda", dtype=torch.float64)
for _ in range(3): a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): a @ b
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("dgemm", f"{ms*1e3:.1f} us", f"{2*M*N*K/ms/1e9:.1f} TFLOP/s")
at = a.t().contiguous()
e0.record()
for _ in range(10): at @ a[:, :256]
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("dgemm atb", f"{ms*1e3:.1f} us")
