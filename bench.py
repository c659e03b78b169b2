#!/usr/bin/env python
"""QPINN train-step collocation points/sec on B200 (BASELINE.json metric).

One "step" = one full training epoch of the reference trainer
(training.py:359-407 without probes): forward with d/dx,y,t tangents
(trunk + K1), the fused Maxwell loss (K4), the full gradient (trunk backward
+ K2 adjoint), [NCCL all-reduce], loss finalisation and Adam.

Workloads: N=1 -> config 2 (vacuum, strongly/acos 7q x 4L, hidden
128, RFF 128, energy + adaptive weighting, 64x64x16 = 2^16 points); N>1 ->
config 3 (128x128x64 = 2^20 points sharded by whole time slices, strong
scaling).  Synthetic = the reference's own seeded init and grid.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--gpus N`` (N > 1) outside torchrun re-executes itself under
``torch.distributed.run`` with N ranks (one per GPU, NCCL, rendezvous on
127.0.0.1); under torchrun WORLD_SIZE must equal N.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QPINN train-step collocation points/sec"
UNIT = "points/s"
WORKLOADS = {
    "config2": dict(grid=(64, 64, 16), name="config2: vacuum 7q x 4L strongly/acos, hidden 128, "
                    "RFF 128, energy + adaptive time weighting, 64x64x16 = 2^16 points"),
    "config3": dict(grid=(128, 128, 64), name="config3: vacuum 7q x 4L strongly/acos, hidden 128, "
                    "RFF 128, energy + adaptive time weighting, 128x128x64 = 2^20 points, "
                    "sharded by time slices"),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=("ours", "reference"))
    p.add_argument("--dtype", default="f32", choices=("f32", "f64"))
    p.add_argument("--workload", default="auto", choices=("auto", "config2", "config3"))
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    return p.parse_args()


def relaunch_distributed(args):
    """``--gpus N`` without a torchrun environment: re-exec under
    torch.distributed.run (N ranks on this node), so ``python bench.py --gpus 8``
    really measures 8 GPUs."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def train_config(grid):
    from paper_2506_23246_b200.network import ModelConfig
    from paper_2506_23246_b200.training import TrainConfig
    return TrainConfig(case="vacuum", model=ModelConfig(variant="hybrid", ansatz="strongly",
                       scale="acos", seed=0), epochs=1, grid=grid, energy_loss_enabled=True,
                       adaptive_weighting=True, eval_cadence=0, probe_cadence=0)


# -- clocks during the timed region ---------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs ~0.1-0.5 s before its first sample: do not
            # start the timed region before it is sampling
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.lines.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def gpu_id_for(dev):
    import torch
    try:
        p = torch.cuda.get_device_properties(dev)
        return f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    except Exception:
        return str(dev)


# -- measured FP32 peak ----------------------------------------------------------------

def fp32_peak():
    import ctypes as C
    from paper_2506_23246_b200 import build as B
    path = B.TOOLS_LIB
    if not os.path.exists(path):
        return None, "unavailable"
    lib = C.CDLL(path)
    a, b, n = C.c_double(), C.c_double(), C.c_int()
    if lib.qpinn_tool_fp32_peak(C.byref(a), C.byref(b), C.byref(n)) != 0:
        return None, "unavailable"
    return max(a.value, b.value), (f"measured in-run: FFMA microbenchmark on {n.value} SMs "
                                   f"(imm {a.value:.1f}, reg {b.value:.1f} TFLOP/s)")


def tensor_gemm_roofline(n_qubits: int, R: int):
    """The transfer map's 3xTF32 tcgen05 GEMM (the forward map Psi = m W':
    [4R, D] x [D, 2D]) timed alone with CUDA events, against cuBLAS's own TF32 peak
    measured in the same run (8192^3, the ceiling for this MMA kind on this box;
    MEASURED_PEAKS.json has bf16 only).  achieved = the TF32 MMA work issued (3
    products) / time."""
    import torch
    from paper_2506_23246_b200 import _native as N
    lib = N.lib()
    M, n, k = 4 * R, 2 << n_qubits, 1 << n_qubits
    A = torch.randn(M, k, device="cuda")
    B = torch.randn(n, k, device="cuda")
    Cm = torch.empty(M, n, device="cuda")
    ws = torch.empty(lib.qpinn_gemm_f32_workspace_bytes(n, k), dtype=torch.uint8, device="cuda")

    def gemm():
        N.check(lib.qpinn_gemm_f32(M, n, k, A.data_ptr(), k, B.data_ptr(), k, Cm.data_ptr(), n,
                                   ws.data_ptr(), ws.numel(), N.stream_ptr()), "gemm")

    def timed(fn, k):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k

    ms = timed(gemm, 20)
    peak = tf32_peak()
    achieved = 3 * 2 * M * n * k / (ms * 1e-3) / 1e12
    return {"bound": "tensor", "achieved": round(achieved, 1), "peak": round(peak, 1),
            "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": None,
            "shape": [M, n, k], "ms_per_launch": round(ms, 4),
            "flop_counting": "TF32 MMA work issued: 3 products x 2 M N K (3xTF32, FP32-class)",
            "peak_source": "measured in-run: cuBLAS TF32 GEMM 8192^3 (torch, allow_tf32)"}


# -- CPU reference (baseline/_ref qpinn, else the oracle port) --------------------------

def _import_reference():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "qpinn")):
        sys.path.insert(0, ref)
        import qpinn  # noqa: F401
        return "reference"
    return "port"


def cpu_reference_rate(grid, seconds, steps=None, warmup=1, sample_slices=1):
    """Time evaluate(tape=True) + adam_step of the reference on a bounded sample
    (the first ``sample_slices`` whole time slices of the workload grid; the
    per-point work equals the full step's)."""
    import numpy as np
    kind = _import_reference()
    cores = os.cpu_count() or 1
    try:
        from threadpoolctl import threadpool_limits
        limiter = threadpool_limits(cores)
    except Exception:  # pragma: no cover
        limiter = None
    rates = []
    if kind == "reference":
        from qpinn.network import ModelConfig, build_model
        from qpinn.physics import (CollocationGrid, LossEvaluator, MaterialMap,
                                   time_bin_weights)
        from qpinn.training import AdamState, adam_step, init_quantum_params
        model = build_model(ModelConfig(variant="hybrid", ansatz="strongly", scale="acos",
                                        seed=0, t_domain=1.5))
        params = model.init_params()
        params.quantum[:] = init_quantum_params("reg", model.n_quantum, 0)
        g = CollocationGrid(*grid, 1.5)
        ev = LossEvaluator(model, g, MaterialMap("vacuum"), case="vacuum", energy_enabled=True,
                           chunk_slices=sample_slices)
        ev.chunks = ev.chunks[:1]
        npts = (ev.chunks[0].s1 - ev.chunks[0].s0) * g.slice_size
        w = np.array([1.0, 0.9, 0.8, 0.7, 0.6])
        adam = AdamState.zeros(model.total_parameter_count)

        def one():
            r = ev.evaluate(params, weights=w, tape=True)
            adam_step(params, r.grad, adam, 1e-3)
    else:
        import oracle as O
        om = O.OracleModel(seed=0)
        flat = om.init_params()
        flat[om.n_classical:] = O.init_quantum_params("reg", om.n_quantum, 0)
        ev = O.Evaluator(om, O.Grid(*grid, 1.5), chunk_slices=sample_slices,
                         slices=list(range(sample_slices)))
        npts = sample_slices * grid[0] * grid[1]
        w = np.array([1.0, 0.9, 0.8, 0.7, 0.6])
        m = np.zeros(om.n_total)
        v = np.zeros(om.n_total)
        st = {"t": 0}

        def one():
            _, grad, _ = ev.evaluate(flat, w, tape=True)
            st["t"] = O.adam_update(flat, grad, m, v, st["t"], 1e-3)
    for _ in range(warmup):
        one()
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        one()
        rates.append(npts / (time.perf_counter() - t0))
        done = len(rates) >= steps if steps else (time.perf_counter() - t_start >= seconds and len(rates) >= 2)
        if done:
            break
    if limiter is not None:
        limiter.unregister() if hasattr(limiter, "unregister") else None
    sample = (f"{sample_slices} whole time slice(s) = {npts} points of the {grid[0]}x{grid[1]}x"
              f"{grid[2]} grid per step, evaluate(tape=True)+adam_step, {len(rates)} timed steps")
    sample += "; value = best step (SURVEY 8d: best of >= 2)"
    return max(rates), kind, cores, sample, rates


# -- our arm --------------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2506_23246_b200 import _native as N
    from paper_2506_23246_b200.training import Trainer, allreduce_fn

    rank, world, local = dist_env()
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    # QPINN_BENCH_FUNCTIONAL_DP=1: functional check of the N>1 path on a one-GPU box
    # (every rank on cuda:0, gloo collectives); its numbers are not bench values
    functional = os.environ.get("QPINN_BENCH_FUNCTIONAL_DP") == "1"
    if functional:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if functional:
            dist.init_process_group("gloo")
        else:
            # NCCL's own log (ranks, NVLink/NVLS transport) goes to stderr so the
            # JSON line stays alone on stdout
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=dev)
    wl = args.workload if args.workload != "auto" else ("config2" if world == 1 else "config3")
    grid = WORKLOADS[wl]["grid"]
    dtype = torch.float32 if args.dtype == "f32" else torch.float64
    cfg = train_config(grid)
    tr = Trainer(cfg, device=dev, dtype=dtype, rank=rank, world_size=world,
                 reduce_fn=allreduce_fn() if world > 1 else None)
    n_total = tr.grid.n_points

    def barrier():
        if world > 1:
            dist.barrier(**({} if functional else {"device_ids": [local]}))

    def timed_steps(k):
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            tr.step()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item())

    for _ in range(max(args.warmup, 3)):
        tr.step()
    launches0 = N.LAUNCHES["count"]
    # clocks are sampled across the three timed passes (value, per-kernel, e2e)
    clk = ClockSampler(gpu_id_for(local)).__enter__()
    ms = timed_steps(args.steps)
    launches = (N.LAUNCHES["count"] - launches0)
    value = n_total * args.steps / (ms / 1e3)

    # per-kernel CUDA-event timing over a second timed pass (own stream = current)
    N.timing(True)
    ms_prof = timed_steps(args.steps)
    kern = N.timer_report()
    N.timing(False)

    # end to end: inputs copied from pinned host memory every step (+ loss D2H)
    tr.set_host_inputs(True)
    for _ in range(2):
        tr.step()
    ms_e2e = timed_steps(args.steps)
    clk.__exit__(None, None, None)
    e2e_value = n_total * args.steps / (ms_e2e / 1e3)
    h2d = tr.host_input_bytes()
    d2h = tr.readback_bytes()

    line = None
    if rank == 0:
        peak, peak_src = fp32_peak()
        circuit = tr.model.circuit
        R_local = tr.evaluator.n_local_points
        rl = roofline_passes(tr, kern, args.steps, ms_prof, dtype, peak, peak_src)
        dom = max(rl, key=lambda k: rl[k]["share_of_step"]) if rl else None
        if circuit.uses_transfer(dtype) and dtype == torch.float32:
            rl["transfer_gemm"] = tensor_gemm_roofline(circuit.n_qubits, R_local)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            v, kind, cores, sample, _ = cpu_reference_rate(grid, args.cpu_seconds)
            cpu = {"value": round(v, 2), "unit": UNIT, "cores": cores, "kind": kind,
                   "sample": sample}
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f32" if dtype == torch.float32 else "f64",
            "data": "synthetic (reference seeded init: Model.init_params + init_quantum_params('reg', 84, 0); reference collocation grid)",
            "config": bench_config(wl, world),
            "e2e": {"value": round(e2e_value, 1), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches),
            "roofline": rl.get(dom) if dom else None,
            "roofline_kernels": rl,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        if functional:
            line["functional_check"] = "all ranks on cuda:0 over gloo: not a bench value"
    if world > 1:
        dist.barrier(**({} if functional else {"device_ids": [local]}))
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


_TF32 = {}


def tf32_peak():
    """cuBLAS TF32 GEMM throughput measured in this run (8192^3, allow_tf32): the
    ceiling of the tensor-core MMA kind our FP32-class GEMMs use.  Dividing by the 3
    products of the 3xTF32 split gives the FP32-class ceiling (MEASURED_PEAKS.json
    carries bf16 only)."""
    if "v" not in _TF32:
        import torch
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = True
        a = torch.randn(8192, 8192, device="cuda")
        b = torch.randn(8192, 8192, device="cuda")
        for _ in range(3):
            a @ b
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            a @ b
        e1.record()
        torch.cuda.synchronize()
        torch.backends.cuda.matmul.allow_tf32 = prev
        _TF32["v"] = 2 * 8192 ** 3 / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e12
    return _TF32["v"]


def roofline_passes(tr, kern, steps, ms_prof, dtype, ffma_peak, ffma_src):
    """Per pass of the step: achieved ALGORITHMIC FLOP/s (SURVEY 8d per-point counts:
    roofline.pqc_flops for the circuit -- the gate-sweep count, whatever formulation
    runs it -- and roofline.trunk_flops for the trunk) over the pass's CUDA-event
    time, against the ceiling of the units that run it:
      * tensor-core passes (the trunk; the transfer-matrix PQC at fp32 n = 5..7):
        the FP32-class ceiling of 3xTF32 = the in-run cuBLAS TF32 peak / 3;
      * CUDA-core passes (the layer-loop PQC kernels): the in-run FFMA peak.
    ``hbm_staged`` is the same pass seen as HBM traffic: the bytes its kernels stage
    through HBM by design (roofline.transfer_bytes / trunk_bytes) and ``traffic`` the
    DRAM bytes ncu measured for it (profiles/traffic.json), per launch."""
    import torch
    from paper_2506_23246_b200.roofline import pqc_flops, transfer_bytes, trunk_bytes, trunk_flops
    circuit = tr.model.circuit
    mc = tr.model.config
    R_local = tr.evaluator.n_local_points
    hbm = hbm_peak()
    transfer = circuit.uses_transfer(dtype)
    f_fwd, f_adj = pqc_flops(circuit)
    t_fwd, t_bwd = trunk_flops(mc.hidden_width, mc.rff_features, mc.n_qubits, tr.model.n_hidden)
    tb_f, tb_b = trunk_bytes(mc.hidden_width, mc.rff_features, mc.n_qubits, tr.model.n_hidden,
                             4 if dtype == torch.float32 else 8)
    pb_f, pb_b = transfer_bytes(circuit.n_qubits) if transfer else (None, None)
    tensor_ceiling = tf32_peak() / 3 if dtype == torch.float32 else None
    spec = {"pqc_forward": (f_fwd, pb_f, transfer), "pqc_backward": (f_adj, pb_b, transfer),
            "trunk_forward": (t_fwd, tb_f, dtype == torch.float32),
            "trunk_backward": (t_bwd, tb_b, dtype == torch.float32)}
    rl = {}
    for name, (flop_pp, bytes_pp, on_tensor) in spec.items():
        if name not in kern:
            continue
        nl, mean_ms = kern[name]
        per_step = nl / steps
        pts = R_local / per_step
        achieved = flop_pp * pts / (mean_ms * 1e-3) / 1e12
        if on_tensor:
            peak, unit_src = tensor_ceiling, ("in-run cuBLAS TF32 GEMM 8192^3 / 3 (the FP32-class "
                                              "ceiling of the 3xTF32 split; MEASURED_PEAKS.json "
                                              "has bf16 only)")
        else:
            peak, unit_src = ffma_peak, ffma_src
        e = {"bound": "tensor" if on_tensor else "fp32", "achieved": round(achieved, 2),
             "peak": round(peak, 1) if peak else None, "unit": "TFLOP/s",
             "frac": round(achieved / peak, 4) if peak else None,
             "traffic": traffic_for(name, pts), "flop_per_point": flop_pp,
             "points_per_launch": pts, "ms_per_launch": round(mean_ms, 4),
             "share_of_step": round(mean_ms * per_step / (ms_prof / steps), 4),
             "peak_source": unit_src,
             "flop_counting": ("SURVEY 8(d) gate-sweep count of the circuit (roofline.pqc_flops)"
                               if name.startswith("pqc") else
                               "SURVEY 8(d) trunk count with tangents (roofline.trunk_flops)")}
        if name.startswith("pqc") and ffma_peak:
            e["fp32_simt_frac"] = round(achieved / ffma_peak, 4)  # north_star's FP32-peak view
        if bytes_pp:
            gbs = bytes_pp * pts / (mean_ms * 1e-3) / 1e9
            e["hbm_staged"] = {"bytes_per_point": bytes_pp, "achieved": round(gbs, 1),
                               "peak": hbm, "unit": "GB/s", "frac": round(gbs / hbm, 4),
                               "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"}
        if name.startswith("pqc"):
            e["path"] = ("transfer matrix (3xTF32 tcgen05 GEMMs)" if transfer
                         else "layer-loop gate sweep (CUDA cores)")
        rl[name] = e
    return rl


def bench_config(wl, world):
    """The workload description, identical for both arms."""
    grid = WORKLOADS[wl]["grid"]
    n = grid[0] * grid[1] * grid[2]
    return {"workload": WORKLOADS[wl]["name"], "points_per_step": n,
            "points_per_gpu": n // world, "grid": list(grid),
            "parallelism": f"dp{world} (whole time slices per rank)",
            "l2": "inputs larger than L2 (per-step activations > 126 MB)"}


def hbm_peak():
    """Measured HBM copy bandwidth (GB/s) from the driver-written MEASURED_PEAKS.json,
    else the B200 profiling recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6500.0


def traffic_for(name, pts):
    """DRAM bytes per launch from the committed ncu capture (profiles/), else None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        per_pt = d[name]["bytes_per_point"]
        return round(per_pt * pts)
    except Exception:
        return None


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    wl = args.workload if args.workload != "auto" else ("config2" if world == 1 else "config3")
    grid = WORKLOADS[wl]["grid"]
    v, kind, cores, sample, rates = cpu_reference_rate(grid, 0, steps=max(args.steps, 2),
                                                       warmup=args.warmup)
    # the whole grid at the sampled per-point rate (a time slice is the sample)
    ms = 1e3 * grid[0] * grid[1] * grid[2] / v
    line = {
        "metric": METRIC, "value": round(v, 2), "unit": UNIT, "n_gpus": world, "impl": "reference",
        "devices": "host CPU cores (the reference has no GPU path); n_gpus is the launch size",
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference seeded init and grid)",
        "config": bench_config(wl, world),
        "host": "numpy/OpenBLAS on the host cores; one whole time slice per timed step",
        "cpu_baseline": {"value": round(v, 2), "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": round(v, 2), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
