"""Config 4: dielectric TEz case across the paper's ansatz x input
scaling ablation grid -- train-step points/s per cell on one B200.

Every cell trains the dielectric model (slab x >= 0.3, eps_r = 4, t_end = 0.7,
diel_balanced, energy term off, y-mirror symmetry) on the 64^3 grid of
configs/dielectric_qpinn.json.  The reference ran cells as independent
processes (cli.py:145-169); on 8 GPUs each cell would be one replica.
Usage: python scripts/sweep_ablation.py [steps] [grid]  -> one JSON line per cell
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_23246_b200.network import ModelConfig  # noqa: E402
from paper_2506_23246_b200.training import TrainConfig, Trainer  # noqa: E402

KINDS = ("basic", "strongly", "cross_mesh", "cross_mesh_2rot", "cross_mesh_cnot", "no_entanglement")
SCALES = ("none", "pi", "bias", "asin", "acos")


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    grid = tuple(int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "64,64,64").split(","))
    for kind in KINDS:
        for scale in SCALES:
            cfg = TrainConfig(case="dielectric", model=ModelConfig(variant="hybrid", ansatz=kind,
                              scale=scale, seed=0), epochs=1, grid=grid, energy_loss_enabled=False,
                              phys_loss_mode="diel_balanced", eval_cadence=0, probe_cadence=0)
            tr = Trainer(cfg, device="cuda", dtype=torch.float32)
            for _ in range(2):
                tr.step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rows = [tr.step() for _ in range(steps)]
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            pts = tr.grid.n_points
            print(json.dumps({"ansatz": kind, "scale": scale, "grid": list(grid), "points": pts,
                              "ms_per_step": round(ms, 3), "points_per_s": round(pts / ms * 1e3),
                              "params": tr.model.total_parameter_count,
                              "loss_first": rows[0].total, "loss_last": rows[-1].total}),
                  flush=True)
            del tr
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
