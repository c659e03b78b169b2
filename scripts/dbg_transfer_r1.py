"""Per-entry errors of the layer and transfer K2 vs the oracle at tiny batches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2506_23246_b200.ansatz import build_circuit, pqc_backward_raw, pqc_forward_raw, state_buffer  # noqa: E402

for R in (1, 65, 1000):
    n, L, kind = 7, 4, "strongly"
    rng = np.random.default_rng(100 + n)
    c0 = build_circuit(kind, n, L)
    d = dict(a=rng.uniform(-0.9, 0.9, (R, n)), da=rng.normal(size=(3, R, n)),
             qp=rng.uniform(0, 2 * np.pi, c0.param_count), gz=rng.normal(size=(R, n)),
             gdz=rng.normal(size=(3, R, n)))
    wg = O.pqc_backward(d["a"], d["da"], d["qp"], kind, "acos", L, d["gz"], d["gdz"])
    for variant in ("layer", "transfer"):
        c = build_circuit(kind, n, L)
        c.set_kernel_variant(variant)
        t = {k: torch.tensor(v, dtype=torch.float32, device="cuda") for k, v in d.items()}
        st = state_buffer(c, t["a"])
        pqc_forward_raw(c, "acos", t["a"], t["da"], t["qp"], st)
        g = pqc_backward_raw(c, "acos", t["a"], t["da"], t["qp"], t["gz"], t["gdz"], st)
        errs = []
        for name, x, w in zip(("ga", "gda", "gq"), g, wg):
            x = x.double().cpu().numpy()
            errs.append(f"{name} abs {np.abs(x - w).max():.2e} rel(max) {np.abs(x - w).max() / np.abs(w).max():.2e}")
        print(R, variant, " | ".join(errs))
