"""SURVEY 8f row 4 measurement: the FDTD reference solver at the paper's
L2-evaluation size (512 x 512, t_end 1.5, 100 snapshots) on one
B200 vs the reference's numpy solver (baseline/_ref) on the host.  Also a
pure stepping rate (no snapshots) in cell-updates/s and the HBM/L2 traffic
model: each step reads Ez, Hx, Hy, eps and writes Ez, Hx, Hy (56 B/cell).
Usage: python scripts/bench_fdtd.py [nx] [cpu: 1|0]  -> JSON lines"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_23246_b200.fdtd import FdtdConfig, _step_plan, run_reference  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 512
do_cpu = (sys.argv[2] != "0") if len(sys.argv) > 2 else True
for case in ("vacuum", "dielectric"):
    cfg = FdtdConfig(nx=nx, ny=nx, case=case, n_snapshots=100)
    dt, steps, snap = _step_plan(cfg)
    run_reference(cfg)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = run_reference(cfg)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0  # includes the D2H copy of all snapshots
    # device-only stepping rate: CUDA events around a snapshot-free run
    cfg_ns = FdtdConfig(nx=nx, ny=nx, case=case, n_snapshots=1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run_reference(cfg_ns)
    e1.record()
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1)
    cells = nx * nx * (steps + 1)
    row = {"case": case, "grid": [nx, nx], "steps": steps, "snapshots": len(snap),
           "gpu_s_with_snapshots_d2h": round(gpu_s, 4), "gpu_ms_stepping": round(dev_ms, 3),
           "cell_updates_per_s": round(cells / (dev_ms / 1e3)),
           "effective_GB_s_56B_per_cell": round(56 * cells / (dev_ms / 1e3) / 1e9, 1)}
    if do_cpu:
        ref_root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "baseline", "_ref")
        sys.path.insert(0, ref_root)
        from qpinn.fdtd import FdtdConfig as RC, run_reference as rr  # noqa: E402
        t0 = time.perf_counter()
        r = rr(RC(nx=nx, ny=nx, case=case, n_snapshots=100))
        cpu_s = time.perf_counter() - t0
        row["cpu_reference_s"] = round(cpu_s, 3)
        row["speedup"] = round(cpu_s / gpu_s, 1)
        row["max_rel_diff_vs_reference"] = float(max(
            np.max(np.abs(getattr(h, k) - getattr(r, k))) / np.max(np.abs(getattr(r, k)))
            for k in ("ez", "hx", "hy")))
    print(json.dumps(row), flush=True)
