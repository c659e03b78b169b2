"""Full train-step repeatability at the bench configuration: two Trainers from the
same initial state run K steps; parameters, Adam moments and loss rows must be
bit-identical after every step.  Usage: race_step.py [steps] [pairs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_23246_b200.training import Trainer  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 30
pairs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = bench.train_config((64, 64, 16))
ref = Trainer(cfg, device="cuda", dtype=torch.float32)
rows_ref, flats = [], []
for _ in range(K):
    rows_ref.append(ref.step().total)
    flats.append(ref.flat.detach().clone())
bad = 0
for pr in range(pairs):
    tr = Trainer(cfg, device="cuda", dtype=torch.float32)
    for k in range(K):
        r = tr.step().total
        if r != rows_ref[k] or not torch.equal(tr.flat, flats[k]):
            bad += 1
            d = (tr.flat - flats[k]).abs()
            print(f"pair {pr} step {k}: loss {r!r} vs {rows_ref[k]!r}, params differ at "
                  f"{int((d != 0).sum())} entries (max {d.max().item():.3e})", flush=True)
            break
print(f"{pairs} repeats of {K} steps: {bad} diverged", flush=True)
