"""Run K1 and K2 alone at config-2 size (R = 2^16, 7q x 4L strongly/acos) for
ncu captures and CUDA-event timing.  Usage: pqc_only.py [R] [kind] [iters] [--variant=layer] [--f64]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_23246_b200.ansatz import (build_circuit, pqc_backward_raw,  # noqa: E402
                                          pqc_forward_raw, state_buffer)
from paper_2506_23246_b200.roofline import pqc_flops  # noqa: E402

pos = [a for a in sys.argv[1:] if not a.startswith("--")]
R = int(pos[0]) if len(pos) > 0 else 1 << 16
kind = pos[1] if len(pos) > 1 else "strongly"
iters = int(pos[2]) if len(pos) > 2 else 20
dtype = torch.float64 if "--f64" in sys.argv else torch.float32
rng = np.random.default_rng(0)
c = build_circuit(kind, 7, 4)
for arg in sys.argv[1:]:
    if arg.startswith("--variant="):  # auto | transfer | layer | generic
        c.set_kernel_variant(arg.split("=", 1)[1])
dev = "cuda"
a = torch.as_tensor(rng.uniform(-0.9, 0.9, (R, 7)), dtype=dtype, device=dev)
da = torch.as_tensor(rng.normal(size=(3, R, 7)), dtype=dtype, device=dev)
qp = torch.as_tensor(rng.uniform(0, 6.28, c.param_count), dtype=dtype, device=dev)
gz = torch.as_tensor(rng.normal(size=(R, 7)), dtype=dtype, device=dev)
gdz = torch.as_tensor(rng.normal(size=(3, R, 7)), dtype=dtype, device=dev)

st = state_buffer(c, a)
for _ in range(3):
    z, dz = pqc_forward_raw(c, "acos", a, da, qp, st)
    pqc_backward_raw(c, "acos", a, da, qp, gz, gdz, st)
torch.cuda.synchronize()
ff, fa = pqc_flops(c)
for name, fn, fl in (("K1 forward+tangent", lambda: pqc_forward_raw(c, "acos", a, da, qp, st), ff),
                     ("K2 adjoint", lambda: pqc_backward_raw(c, "acos", a, da, qp, gz, gdz, st), fa),
                     ("K2 adjoint (replay, no hand-off)",
                      lambda: pqc_backward_raw(c, "acos", a, da, qp, gz, gdz), fa)):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"{name}: {ms:.4f} ms  {fl * R / ms / 1e9:.2f} TFLOP/s algorithmic")
