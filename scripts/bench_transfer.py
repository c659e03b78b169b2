"""K1/K2 timing: layer-loop kernels vs the transfer-matrix path (n = 7, L = 4, 2^16 points)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_23246_b200.ansatz import (build_circuit, pqc_backward_raw, pqc_forward_raw,  # noqa: E402
                                          state_buffer)

R = int(os.environ.get("R", 65536))
for n in (int(v) for v in os.environ.get("NS", "7").split(",")):
    for kind in os.environ.get("KINDS", "strongly,cross_mesh").split(","):
        for variant in os.environ.get("VARIANTS", "auto,transfer").split(","):
            c = build_circuit(kind, n, 4)
            c.set_kernel_variant(variant)
            g = torch.Generator(device="cuda").manual_seed(0)
            a = torch.rand((R, n), device="cuda", generator=g) * 1.8 - 0.9
            da = torch.randn((3, R, n), device="cuda", generator=g)
            qp = torch.rand(c.param_count, device="cuda", generator=g) * 6.28
            gz = torch.randn((R, n), device="cuda", generator=g)
            gdz = torch.randn((3, R, n), device="cuda", generator=g)
            st = state_buffer(c, a)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            for _ in range(3):
                pqc_forward_raw(c, "acos", a, da, qp, st)
                pqc_backward_raw(c, "acos", a, da, qp, gz, gdz, st)
            tf = tb = 0.0
            K = int(os.environ.get("K", 20))
            for _ in range(K):
                ev[0].record()
                pqc_forward_raw(c, "acos", a, da, qp, st)
                ev[1].record()
                pqc_backward_raw(c, "acos", a, da, qp, gz, gdz, st)
                ev[2].record()
                torch.cuda.synchronize()
                tf += ev[0].elapsed_time(ev[1])
                tb += ev[1].elapsed_time(ev[2])
            print(f"n={n} {kind:12s} {variant:9s} fwd {tf / K * 1e3:7.1f} us  bwd {tb / K * 1e3:7.1f} us",
                  flush=True)
