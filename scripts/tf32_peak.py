import torch
torch.backends.cuda.matmul.allow_tf32 = True
for dt, name in ((torch.float32, "tf32"), (torch.bfloat16, "bf16")):
    for n in (8192,):
        a = torch.randn(n, n, device="cuda", dtype=dt); b = torch.randn(n, n, device="cuda", dtype=dt)
        for _ in range(3): a @ b
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): a @ b
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(name, n, f"{2 * n**3 / ms / 1e9:.0f} TFLOP/s")
# our shape with cuBLAS tf32
M, N, K = 262144, 256, 256
a = torch.randn(M, K, device="cuda"); b = torch.randn(K, N, device="cuda")
for _ in range(3): a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): a @ b
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print("cublas tf32 262144x256x256", f"{ms*1e3:.1f} us", f"{2*M*N*K/ms/1e9:.0f} TFLOP/s")
