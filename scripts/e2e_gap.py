"""Where the e2e step's extra time goes: device-timed steps in the device-resident
mode and in the host-input mode, plus host-side time per step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_23246_b200.training import Trainer  # noqa: E402

cfg = bench.train_config((64, 64, 16))
tr = Trainer(cfg, device="cuda", dtype=torch.float32)
for _ in range(5):
    tr.step()


def timed(k):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(k):
        tr.step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k, (time.perf_counter() - t0) * 1e3 / k


order = sys.argv[1].split(",") if len(sys.argv) > 1 else ["device", "host", "device", "host"]
for mode in order:
    tr.set_host_inputs(mode == "host")
    for _ in range(3):
        tr.step()
    print(mode, "ms/step device %.4f  host %.4f" % timed(50), flush=True)
