"""One eager training step (config 2) between cudaProfilerStart/Stop, for
    ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,...
The per-kernel DRAM bytes become profiles/traffic.json (bytes per point per pass)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import WORKLOADS, train_config  # noqa: E402
from paper_2506_23246_b200.training import Trainer  # noqa: E402

tr = Trainer(train_config(WORKLOADS["config2"]["grid"]), device="cuda", dtype=torch.float32,
             graphs=False)
for _ in range(3):
    tr.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
tr.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("points", tr.grid.n_points)
