"""One transfer-path forward (with tangents) at R points, for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_23246_b200.ansatz import build_circuit, pqc_forward_raw  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
tan = len(sys.argv) <= 2 or sys.argv[2] != "notan"
rng = np.random.default_rng(5)
a = torch.as_tensor(rng.uniform(-0.95, 0.95, (R, 7)), dtype=torch.float32, device="cuda")
da = torch.as_tensor(rng.normal(size=(3, R, 7)), dtype=torch.float32, device="cuda")
c = build_circuit("strongly", 7, 4)
qp = torch.as_tensor(rng.uniform(0, 6.28, c.param_count), dtype=torch.float32, device="cuda")
z, dz = pqc_forward_raw(c, "acos", a, da if tan else None, qp)
torch.cuda.synchronize()
print("ok", float(z.abs().sum()))
