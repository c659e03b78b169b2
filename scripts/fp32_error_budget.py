"""FP32 error budget of Model.forward at the bench configuration, stage by stage.

Runs on the GPU box.  The bench model (7q x 4L strongly/acos, hidden 128, RFF
128) at its reference initial parameters (tests/golden/step_headline.npz) on
the first two time slices of the 64x64x16 grid.  The float64 build is the
reference (it matches the reference to ~1e-15, tests/test_headline_gpu.py).

For each stage the table gives max|err| / max|ref|:
* floor  : the float64 computation on float32-ROUNDED inputs -- what any
           FP32 implementation inherits before doing arithmetic;
* fp32   : our float32 kernels on the same rounded inputs (own error);
* chain  : float32 end to end (errors of earlier stages propagated).

    python scripts/fp32_error_budget.py  [> profiles/r02/fp32_error_budget.json]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2506_23246_b200.ansatz import BatchedDual, quantum_layer_forward  # noqa: E402
from paper_2506_23246_b200.network import Model, ModelConfig  # noqa: E402
from paper_2506_23246_b200.physics import CollocationGrid  # noqa: E402


def rel(a, b):
    a = a.double().cpu().numpy() if torch.is_tensor(a) else np.asarray(a)
    b = b.double().cpu().numpy() if torch.is_tensor(b) else np.asarray(b)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def main():
    g = np.load(os.path.join(ROOT, "tests", "golden", "step_headline.npz"))
    cfg = ModelConfig(variant="hybrid", ansatz="strongly", scale="acos", seed=0, t_domain=1.5)
    m64 = Model(cfg, device="cuda", dtype=torch.float64)
    m32 = Model(cfg, device="cuda", dtype=torch.float32)
    p64 = m64.params_from(g["flat0"])
    p32 = m32.params_from(g["flat0"])
    n = int(g["forward_points"])
    x, y, t = CollocationGrid(64, 64, 16, 1.5).flat_points()
    x, y, t = x[:n], y[:n], t[:n]
    out = {}

    def adapter(model, params):
        v = model.views(params.flat)
        X, Y, T = model._coords(x, y, t)
        h, dh = model.trunk(v, X, Y, T, True)
        a = torch.tanh(h @ v["adapter.W"] + v["adapter.b"])
        da = (1.0 - a * a) * (dh @ v["adapter.W"])
        return a, da, v

    a64, da64, v64 = adapter(m64, p64)
    a32, da32, v32 = adapter(m32, p32)
    out["trunk+adapter a  (chain)"] = rel(a32, a64)
    out["trunk+adapter da (chain)"] = rel(da32, da64)
    circ64, circ32 = m64.circuit, m32.circuit
    q64, q32 = v64["quantum"], v32["quantum"]

    def pqc(circ, a, da, qp):
        r = quantum_layer_forward(BatchedDual(a, da), qp, circ, "acos", check=False)
        return r.val, r.tan

    z64, dz64 = pqc(circ64, a64, da64, q64)
    r = lambda v: v.float().double()  # noqa: E731
    zf, dzf = pqc(circ64, r(a64), r(da64), r(q64))
    out["pqc z  floor"] = rel(zf, z64)
    out["pqc dz floor"] = rel(dzf, dz64)
    for variant in ("transfer", "layer"):
        circ32.set_kernel_variant(variant)
        z32, dz32 = pqc(circ32, a64.float(), da64.float(), q32)
        out[f"pqc z  fp32 [{variant}]"] = rel(z32, z64)
        out[f"pqc dz fp32 [{variant}]"] = rel(dz32, dz64)
        zc, dzc = pqc(circ32, a32, da32, q32)
        out[f"pqc z  chain [{variant}]"] = rel(zc, z64)
        out[f"pqc dz chain [{variant}]"] = rel(dzc, dz64)
    circ32.set_kernel_variant("auto")
    f64_, j64 = m64.forward(p64, x, y, t, derivs=True)
    f32_, j32 = m32.forward(p32, x, y, t, derivs=True)
    F64 = torch.stack([f64_.ez, f64_.hx, f64_.hy])
    F32 = torch.stack([f32_.ez, f32_.hx, f32_.hy])
    J64 = torch.stack([j64.ez, j64.hx, j64.hy])
    J32 = torch.stack([j32.ez, j32.hx, j32.hy])
    out["fields (chain)"] = rel(F32, F64)
    out["jacobians (chain)"] = rel(J32, J64)
    out["fields f64 vs reference golden"] = rel(F64, g["fields"])
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
