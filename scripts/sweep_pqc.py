"""Config 5: standalone PQC forward+tangent (K1) and adjoint (K2)
sweep over n = 4..16 qubits, L in {1, 4, 8} layers and batch sizes, for the
three entangler families (strongly: CNOT permutation, cross_mesh: CRZ phase
diagonal, no_entanglement), acos scaling.

Inputs: a ~ U(-0.9, 0.9) [R,n], tangents ~ N(0,1) [3,R,n], qparams ~ U(0, 2pi),
seed 0.  R*2^n is capped (the statevector work per point grows as 2^n); the
metric is points/s and algorithmic TFLOP/s (roofline.pqc_flops).
Usage: python scripts/sweep_pqc.py [--quick] [--n=..] [--variant=..] [--all-ansatze]   -> one JSON line per cell
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_23246_b200 import CapacityError  # noqa: E402
from paper_2506_23246_b200.ansatz import (build_circuit, pqc_backward_raw, pqc_forward_raw,  # noqa: E402
                                          state_buffer)
from paper_2506_23246_b200.roofline import pqc_flops  # noqa: E402


def time_fn(fn, min_s=0.05, max_iter=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 1
    while True:
        e0.record()
        for _ in range(it):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if ms / 1e3 >= min_s or it >= max_iter:
            return ms / it
        it = min(max_iter, it * 4)


def main():
    quick = "--quick" in sys.argv
    rng = np.random.default_rng(0)
    ns = range(4, 17)
    variant = None
    for arg in sys.argv[1:]:
        if arg.startswith("--n="):  # e.g. --n=15,16
            ns = [int(v) for v in arg[4:].split(",")]
        if arg.startswith("--variant="):  # auto | transfer | layer | generic
            variant = arg.split("=", 1)[1]
    Ls = (1, 4) if quick else (1, 4, 8)
    kinds = ("strongly", "cross_mesh", "no_entanglement")
    if "--all-ansatze" in sys.argv:  # all six ansatze
        kinds = ("basic", "strongly", "cross_mesh", "cross_mesh_2rot", "cross_mesh_cnot",
                 "no_entanglement")
    for n in ns:
        for L in Ls:
            for kind in kinds:
                # batch: 2^16 (2^20 for n <= 8) capped so that R * 2^n <= 2^24 (n > 8: <= 2^26)
                R = (1 << 20) if n <= 8 else (1 << 16)
                R = min(R, (1 << (24 if n <= 8 else 26)) >> n) if n > 8 else R
                if quick:
                    R = min(R, 1 << 14)
                # layer-boundary hand-off (n <= 8): 4 states x 2^n x L per row, keep <= 4 GiB
                if n <= 8:
                    R = min(R, (4 << 30) // (L * 4 * (1 << n) * 8))
                c = build_circuit(kind, n, L)
                if variant:
                    c.set_kernel_variant(variant)
                a = torch.as_tensor(rng.uniform(-0.9, 0.9, (R, n)), dtype=torch.float32, device="cuda")
                da = torch.as_tensor(rng.normal(size=(3, R, n)), dtype=torch.float32, device="cuda")
                qp = torch.as_tensor(rng.uniform(0, 2 * np.pi, c.param_count), dtype=torch.float32,
                                     device="cuda")
                g = torch.randn_like(a)
                gd = torch.randn_like(da)
                ff, fa = pqc_flops(c)
                row = {"n": n, "L": L, "ansatz": kind, "R": R, "params": c.param_count}
                st = state_buffer(c, a) if n <= 8 else None
                ms_f = time_fn(lambda: pqc_forward_raw(c, "acos", a, da, qp, st))
                row["k1_ms"] = round(ms_f, 4)
                row["k1_points_per_s"] = round(R / ms_f * 1e3)
                row["k1_tflops"] = round(ff * R / ms_f / 1e9, 2)
                try:
                    ms_b = time_fn(lambda: pqc_backward_raw(c, "acos", a, da, qp, g, gd, st))
                    row["k2_ms"] = round(ms_b, 4)
                    row["k2_points_per_s"] = round(R / ms_b * 1e3)
                    row["k2_tflops"] = round(fa * R / ms_b / 1e9, 2)
                except CapacityError as e:
                    row["k2"] = f"unsupported: {e}"
                row["regime"] = c.regime(torch.float32)  # K1's kernels (qpinn_pqc_regime)
                row["k2_regime"] = c.regime(torch.float32, backward=True)
                print(json.dumps(row), flush=True)
                del a, da, g, gd, st
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
