"""Repeat the transfer-path PQC forward (with and without tangents) and the bench
step's forward, comparing every repeat bitwise with the first: any difference is
a race.  Usage: race_check.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_23246_b200.ansatz import build_circuit, pqc_forward_raw  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rng = np.random.default_rng(5)
R, n, L = 1 << 16, 7, 4
dev = "cuda"
a = torch.as_tensor(rng.uniform(-0.95, 0.95, (R, n)), dtype=torch.float32, device=dev)
da = torch.as_tensor(rng.normal(size=(3, R, n)), dtype=torch.float32, device=dev)
for kind in ("strongly", "no_entanglement"):
    c = build_circuit(kind, n, L)
    qp = torch.as_tensor(rng.uniform(0, 2 * np.pi, c.param_count), dtype=torch.float32, device=dev)
    for tan in (True, False):
        ref = None
        bad = 0
        for r in range(reps):
            z, dz = pqc_forward_raw(c, "acos", a, da if tan else None, qp)
            out = torch.cat([z.flatten()] + ([dz.flatten()] if tan else []))
            if ref is None:
                ref = out.clone()
                continue
            if not torch.equal(out, ref):
                bad += 1
                d = (out - ref).abs()
                idx = torch.nonzero(d).flatten()
                print(f"{kind} tan={tan} rep {r}: {idx.numel()} entries differ, max {d.max().item():.3e}, "
                      f"first flat idx {idx[:8].tolist()}", flush=True)
        print(f"{kind} tan={tan}: {bad}/{reps - 1} repeats differ", flush=True)
