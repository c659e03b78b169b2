import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2506_23246_b200 import _native as N
lib = N.lib()
rows, m, n = 64, 128, 128
X = torch.ones(rows, m, device="cuda"); G = torch.ones(rows, n, device="cuda")
X[:, 1] = 2.0; G[:, 3] = 3.0
C = torch.full((m, n), -7.0, device="cuda")
wsb = lib.qpinn_gemm_f32_atb_workspace_bytes(rows, m, n)
ws = torch.full((wsb // 4,), -5.0, device="cuda")
rc = lib.qpinn_gemm_f32_atb(rows, m, n, X.data_ptr(), m, G.data_ptr(), n, C.data_ptr(), ws.data_ptr(), wsb, N.stream_ptr())
torch.cuda.synchronize()
print("rc", rc, lib.qpinn_last_error())
print("C", C[0, :6].tolist(), C[1, :6].tolist(), C[5, 2:5].tolist())
p = ws[0:m * n].view(m, n)
print("partial0", p[0, :6].tolist())
print("nonzero partial entries", (ws != 0).sum().item(), "of", ws.numel(), "untouched", (ws == -5).sum().item())
print("raw A first float4s", ws[8192: 8192 + 16].tolist())
print("raw B first float4s", ws[8192 + 512: 8192 + 512 + 16].tolist())
print("acc0 per m", ws[0:8].tolist())
