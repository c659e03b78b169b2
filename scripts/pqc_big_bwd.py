"""One large-n K2 call (adjoint) for ncu / timing: pqc_big_bwd.py n L R [kind]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_23246_b200.ansatz import build_circuit, pqc_backward_raw  # noqa: E402
from paper_2506_23246_b200.roofline import pqc_flops  # noqa: E402

n, L, R = (int(v) for v in sys.argv[1:4])
kind = sys.argv[4] if len(sys.argv) > 4 else "strongly"
rng = np.random.default_rng(0)
c = build_circuit(kind, n, L)
t = lambda *s: torch.as_tensor(rng.normal(size=s), dtype=torch.float32, device="cuda")  # noqa: E731
a = torch.as_tensor(rng.uniform(-0.9, 0.9, (R, n)), dtype=torch.float32, device="cuda")
da, gz, gdz = t(3, R, n), t(R, n), t(3, R, n)
qp = torch.as_tensor(rng.uniform(0, 6.28, c.param_count), dtype=torch.float32, device="cuda")
pqc_backward_raw(c, "acos", a, da, qp, gz, gdz)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
pqc_backward_raw(c, "acos", a, da, qp, gz, gdz)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"K2 n={n} L={L} R={R} {kind}: {ms:.3f} ms, {pqc_flops(c)[1] * R / ms / 1e9:.2f} TFLOP/s")
