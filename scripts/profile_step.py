"""Per-kernel GPU time of one config-2 train step via torch.profiler (CUPTI)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2506_23246_b200.training import Trainer  # noqa: E402

grid = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "64,64,16").split(","))
dtype = torch.float64 if "--f64" in sys.argv else torch.float32
tr = Trainer(bench.train_config(grid), device="cuda", dtype=dtype)
for _ in range(3):
    tr.step()
torch.cuda.synchronize()
steps = 5
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(steps):
        tr.step()
    torch.cuda.synchronize()
ka = prof.key_averages()
rows = []
for e in ka:
    t = getattr(e, "device_time_total", None) or getattr(e, "cuda_time_total", 0)
    if t and e.device_type == torch.autograd.DeviceType.CUDA:
        rows.append((t / steps, e.count // steps, e.key))
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
print(f"GPU kernel time per step: {tot/1000:.3f} ms over {sum(r[1] for r in rows)} launches")
for t, c, k in rows[:40]:
    print(f"{t/1000:8.3f} ms {100*t/tot:5.1f}%  x{c:3d}  {k[:110]}")
