"""Parity at the sizes bench.py times (VERDICT r1 "next round" item 1).

* SURVEY 8(d) config 2, the bench workload: vacuum strongly/acos 7q x 4L,
  hidden 128, RFF 128, energy + adaptive weighting, 64x64x16 = 2^16 points.
  ``Trainer`` is built exactly as ``bench.py`` builds it (fp32 transfer-matrix
  PQC on the tcgen05 GEMMs, default chunking, CUDA graphs on: epoch 0 eager,
  epoch 1 captured, epoch 2 replayed) and its first three epochs are compared
  with the reference trainer's (``tests/golden/make_golden_r2.py``): the
  untaped-pass bin weights, every epoch's loss breakdown and full 66,932-entry
  gradient, the parameters after three Adam steps, and Model.forward fields
  + jacobians on two whole time slices.
* the same model on the 8x8x8 grid, 1000 Adam epochs,
  loss curve vs the reference trainer (pointwise up to the run's chaos onset,
  measured from the reference's own sensitivity; best-so-far loss after it).

Error budget (stated per quantity; ``QPINN_PARITY_REPORT=<dir>`` also writes
the measured errors as JSON):
* FP64 verification build: 1e-10 relative everywhere (north_star), final
  parameters after 3 / 1000 Adam steps within 1e-9 / 1e-8 absolute.
* FP32: loss terms and bin weights |got - want| <= 1e-5 |want| + 1e-6
  max|want| (the SURVEY 8.C FP32 parity definition); the flat gradient and
  Model.forward's fields / jacobians <= 1e-5 norm-relative (north_star's 1e-5
  on the vector; SURVEY 8.C's alternative definition -- elementwise errors and
  their input-rounding floors are in the report and
  scripts/fp32_error_budget.py); the curve <= 1e-4 relative before the chaos
  onset (a 1e-7 perturbation moves it by ~1e-6 there).
"""
import json
import os

import numpy as np
import pytest
import torch

from conftest import load_golden
from gpu_util import assert_close

pytestmark = pytest.mark.gpu


def errors(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    d = np.abs(got - want)
    scale = max(np.max(np.abs(want)), 1e-300)
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(np.abs(want) > 0, d / np.abs(want), np.where(d > 0, np.inf, 0.0))
    return {"norm_rel": float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)),
            "max_abs_over_max": float(np.max(d) / scale),
            "worst_elem_rel": float(np.max(rel)),
            "frac_elem_rel_gt_1e-5": float(np.mean(rel > 1e-5))}


def report(name, rows):
    d = os.environ.get("QPINN_PARITY_REPORT")
    print(name, json.dumps(rows, indent=1))
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, name + ".json"), "w") as f:
            json.dump(rows, f, indent=1)


def bench_config(grid, epochs=1):
    """bench.py's train_config(grid)."""
    from paper_2506_23246_b200.network import ModelConfig
    from paper_2506_23246_b200.training import TrainConfig
    return TrainConfig(case="vacuum", model=ModelConfig(variant="hybrid", ansatz="strongly",
                       scale="acos", seed=0), epochs=epochs, grid=grid,
                       energy_loss_enabled=True, adaptive_weighting=True, eval_cadence=0,
                       probe_cadence=0)


def bench_trainer(dtype, grid):
    """... and bench.py's Trainer(cfg, dtype=...) defaults."""
    from paper_2506_23246_b200.training import Trainer
    cfg = bench_config(grid)
    return cfg, Trainer(cfg, device="cuda", dtype=dtype)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["f32", "f64"])
def test_headline_steps_match_reference(dtype):
    """Kernel parity on the bench path at every epoch: before epoch e the
    trainer's parameters and bin weights are set (in place, so the captured
    graph sees them) to the reference trainer's epoch-e values; the epoch's
    gradient and loss breakdown are then compared."""
    g = load_golden("step_headline.npz")
    f64 = dtype == torch.float64
    _, tr = bench_trainer(dtype, (64, 64, 16))
    assert tr.evaluator.n_local_points == 65536
    if dtype == torch.float32:
        assert tr.model.circuit.uses_transfer(dtype), "the bench path is the transfer path"
    assert np.array_equal(tr.flat.detach().double().cpu().numpy(),
                          g["flat0"].astype(np.float32 if not f64 else np.float64))
    rows = {"chunks": len(tr.evaluator.chunks), "graphs": tr.use_graphs}
    w0 = tr.weights.cpu().numpy()
    rows["weights0 (untaped pass)"] = errors(w0, g["weights"][0])
    assert_close(w0, g["weights"][0], dtype, "bin weights from the untaped pass")
    q = tr.model.n_classical
    bds, bins = [], []
    for e in range(3):
        with torch.no_grad():
            tr.flat.copy_(torch.as_tensor(g["flat"][e], dtype=dtype))
            tr.weights.copy_(torch.as_tensor(g["weights"][e], dtype=torch.float64))
        row = tr.step()
        bd = np.array([row.phys, row.ic, row.sym, row.energy, row.total])
        grad = tr.grad.detach().double().cpu().numpy()
        bds.append(bd)
        bins.append(np.array(row.bin_phys))
        rows[f"breakdown{e}"] = errors(bd, g["breakdown"][e])
        rows[f"bin_phys{e}"] = errors(row.bin_phys, g["bin_phys"][e])
        rows[f"grad{e}"] = errors(grad, g["grad"][e])
        rows[f"grad{e}_quantum"] = errors(grad[q:], g["grad"][e][q:])
        rows[f"grad{e}_classical"] = errors(grad[:q], g["grad"][e][:q])
    rows["graph_replayed"] = bool(tr._graphs)
    report(f"headline_{'f64' if f64 else 'f32'}", rows)
    assert rows["graph_replayed"]
    for e in range(3):
        assert_close(bds[e], g["breakdown"][e], dtype, f"loss breakdown, epoch {e}")
        assert_close(bins[e], g["bin_phys"][e], dtype, f"bin_phys, epoch {e}")
        assert rows[f"grad{e}"]["norm_rel"] <= (1e-10 if f64 else 1e-5), rows[f"grad{e}"]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["f32", "f64"])
def test_headline_free_running_three_epochs(dtype):
    """The bench flow untouched for three epochs: losses vs the reference
    trainer, and where the parameters end up."""
    g = load_golden("step_headline.npz")
    f64 = dtype == torch.float64
    _, tr = bench_trainer(dtype, (64, 64, 16))
    rows, bds = {}, []
    for e in range(3):
        row = tr.step()
        bds.append(np.array([row.phys, row.ic, row.sym, row.energy, row.total]))
        rows[f"breakdown{e}"] = errors(bds[-1], g["breakdown"][e])
    flat = tr.flat.detach().double().cpu().numpy()
    dw, dg = flat - g["flat0"], g["final_flat"] - g["flat0"]
    rows["final_flat_max_abs"] = float(np.max(np.abs(flat - g["final_flat"])))
    rows["update_norm_rel"] = float(np.linalg.norm(dw - dg) / np.linalg.norm(dg))
    report(f"headline_free_{'f64' if f64 else 'f32'}", rows)
    for e in range(3):
        assert_close(bds[e], g["breakdown"][e], dtype, f"loss breakdown, epoch {e}")
    if f64:
        assert rows["final_flat_max_abs"] <= 1e-9
    else:
        # Adam divides each entry by its own running magnitude: entries whose
        # gradient is at rounding level in both builds move by up to lr either
        # way (measured: max 2.5e-3 = 2.5 lr after 3 steps), so the update
        # vector is compared in norm
        assert rows["update_norm_rel"] <= 0.05, rows["update_norm_rel"]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["f32", "f64"])
def test_headline_model_forward(dtype):
    """Model.forward (network.py:284-308) fields + jacobians on two whole time
    slices of the bench grid at the reference initial parameters."""
    g = load_golden("step_headline.npz")
    from paper_2506_23246_b200.network import Model, ModelConfig
    from paper_2506_23246_b200.physics import CollocationGrid
    model = Model(ModelConfig(variant="hybrid", ansatz="strongly", scale="acos", seed=0,
                              t_domain=1.5), device="cuda", dtype=dtype)
    x, y, t = CollocationGrid(64, 64, 16, 1.5).flat_points()
    n = int(g["forward_points"])
    fields, derivs = model.forward(model.params_from(g["flat0"]), x[:n], y[:n], t[:n],
                                   derivs=True)
    fz = torch.stack([fields.ez, fields.hx, fields.hy]).double().cpu().numpy()
    dz = torch.stack([derivs.ez, derivs.hx, derivs.hy]).double().cpu().numpy()
    rows = {"fields": errors(fz, g["fields"]), "derivs": errors(dz, g["derivs"])}
    report(f"headline_forward_{'f64' if dtype == torch.float64 else 'f32'}", rows)
    if dtype == torch.float64:
        assert_close(fz, g["fields"], dtype, "Model.forward fields")
        assert_close(dz, g["derivs"], dtype, "Model.forward jacobians")
    else:  # the whole chain: norm-relative, elementwise in the report
        assert rows["fields"]["norm_rel"] <= 1e-5 and rows["derivs"]["norm_rel"] <= 1e-5, rows


def pointwise_window(g, margin=32):
    """Epochs compared pointwise: up to ``margin`` epochs before the reference's
    first loss rise (its first Adam loss spike, epoch 453).  From the spike on
    the training trajectory is chaotic: the reference restarted from a
    1e-15-relative perturbation of its initial parameters stays within 5e-14 of
    itself until epoch 440 and then drifts by up to 0.4 relative
    (train_config1_sens_1e-15.npz; 1e-7: train_config1_sens_1e-07.npz)."""
    up = np.flatnonzero(g[1:] > 1.01 * g[:-1]) + 1
    return int(up[0]) - margin if up.size else len(g)


def runmin_log_dev(a, b):
    """max |log10 min_{e'<=e} a - log10 min_{e'<=e} b| over e (best-so-far losses)."""
    return np.abs(np.log10(np.minimum.accumulate(a)) - np.log10(np.minimum.accumulate(b)))


@pytest.mark.parametrize("dtype,rtol,chaos_tol", [(torch.float64, 1e-9, 0.05),
                                                  (torch.float32, 1e-4, 0.25)],
                         ids=["f64", "f32"])
def test_config1_curve_1k_steps(dtype, rtol, chaos_tol):
    """7q x 4L on 8x8x8, 1000 Adam epochs of training.train.

    The reference's own run is chaotic from its first Adam loss spike (epoch
    453) on: restarted from a 1e-15-relative perturbation of its initial
    parameters it stays within 5e-14 of itself up to epoch 440 and then drifts
    by up to 0.4 relative (train_config1_sens_1e-15.npz).  So the curve is
    compared pointwise (rtol) up to 32 epochs before that spike, and over the
    whole run by the best-so-far loss in log10 (``chaos_tol``; the reference's
    own 1e-15 / 1e-7 perturbations give 0.011 / 0.027) and the best loss of the
    last 100 epochs."""
    from paper_2506_23246_b200.training import train
    g = load_golden("train_config1.npz")
    sens = load_golden("train_config1_sens_1e-15.npz")["total"]
    sens7 = load_golden("train_config1_sens_1e-07.npz")["total"]
    onset = pointwise_window(g["total"])
    assert 100 <= onset < 1000, onset
    cfg = bench_config((8, 8, 8), epochs=1000)
    res = train(cfg, dtype=dtype)
    rows = {"pointwise_window_epochs": onset}
    for k in ("total", "phys", "ic", "sym", "energy"):
        got = np.array([getattr(r, k) for r in res.log.rows])
        rel = np.abs(got - g[k]) / np.abs(g[k])
        rows[k] = {"max_rel_before_onset": float(rel[:onset].max()),
                   "max_rel_after_onset": float(rel[onset:].max())}
    tot = np.array([r.total for r in res.log.rows])
    rows["runmin_log10_dev_after_onset"] = float(runmin_log_dev(tot, g["total"])[onset:].max())
    rows["reference_self_runmin_log10_dev_1e-15"] = float(
        runmin_log_dev(sens, g["total"])[onset:].max())
    rows["reference_self_runmin_log10_dev_1e-07"] = float(
        runmin_log_dev(sens7, g["total"])[onset:].max())
    rows["final100_min_ratio"] = float(tot[-100:].min() / g["total"][-100:].min())
    flat = res.params.flat.detach().double().cpu().numpy()
    rows["final_flat_max_abs"] = float(np.max(np.abs(flat - g["final_flat"])))
    rows["loss_drop"] = float(g["total"][0] / g["total"][-1])
    rows["curve"] = [float(v) for v in tot]
    report(f"config1_curve_{'f64' if dtype == torch.float64 else 'f32'}", rows)
    assert rows["total"]["max_rel_before_onset"] <= rtol, rows["total"]
    assert rows["runmin_log10_dev_after_onset"] <= chaos_tol, rows["runmin_log10_dev_after_onset"]
    lo, hi = (0.99, 1.01) if dtype == torch.float64 else (0.7, 1.4)
    assert lo <= rows["final100_min_ratio"] <= hi, rows["final100_min_ratio"]


def test_model_forward_runs_our_kernels_only():
    """Model.forward(derivs=True) in fp32 launches no library GEMM (cuBLAS /
    CUTLASS): the trunk, the PQC and the head are this repo's kernels."""
    import re
    from torch.profiler import ProfilerActivity, profile
    from paper_2506_23246_b200.network import Model, ModelConfig
    model = Model(ModelConfig(variant="hybrid", ansatz="strongly", scale="acos", seed=0,
                              t_domain=1.5), device="cuda", dtype=torch.float32)
    p = model.init_params()
    rng = np.random.default_rng(0)
    x, y, t = (torch.as_tensor(v, dtype=torch.float32, device="cuda") for v in
               (rng.uniform(-1, 1, 4096), rng.uniform(-1, 1, 4096), rng.uniform(0, 1.5, 4096)))
    model.forward(p, x, y, t, derivs=True)  # warm (circuit plan upload, weight split)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        model.forward(p, x, y, t, derivs=True)
        torch.cuda.synchronize()
    names = [e.key for e in prof.key_averages()]
    lib = [k for k in names if re.search(r"cublas|cutlass|sgemm|dgemm|xmma|gemv|splitK|nvjet",
                                         k, re.I)]
    assert not lib, f"library GEMM kernels in Model.forward: {lib}"
    ours = [k for k in names if re.search(r"gemm3_kernel|pqc|tr_|features|head", k)]
    assert any("gemm3_kernel" in k for k in ours), names


def test_bench_steps_bitwise_repeatable():
    """Two bench trainers from the same initial state stay bit-identical over 15
    steps (graph replays included): no data race anywhere in the step
    (scripts/race_step.py runs the longer version)."""
    _, a = bench_trainer(torch.float32, (64, 64, 16))
    _, b = bench_trainer(torch.float32, (64, 64, 16))
    for _ in range(15):
        ra, rb = a.step(), b.step()
        assert ra.total == rb.total
        assert torch.equal(a.flat, b.flat)
