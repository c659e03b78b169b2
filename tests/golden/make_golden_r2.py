"""Golden vectors at the bench's own sizes, generated from the reference itself.

Run in the build container (the reference is importable only here):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_r2.py [step|curve|all]

Fixtures
--------
step_headline.npz  SURVEY 8(d) config 2, the configuration bench.py times:
                   vacuum, strongly/acos 7q x 4L, hidden 128, RFF 128, energy +
                   adaptive time weighting, 64x64x16 = 2^16 points, t_end 1.5.
                   The first three epochs of the reference trainer
                   (training.py:309-414), replayed step by step with the
                   reference's own LossEvaluator / time_bin_weights / adam_step
                   so that every epoch's parameters, full 66,932-entry gradient,
                   breakdown and bin weights are recorded (train() does not expose
                   the gradient).
                   Also Model.forward (network.py:284-308) fields + jacobians on
                   the first two time slices.
train_config1.npz  SURVEY 8(d) config 1: the vacuum_qpinn.json model (7q x 4L,
                   hidden 128, RFF 128) on the 8x8x8 grid, 1000 epochs of
                   training.train: per-epoch loss terms and the final parameters.
train_config1_sens_<rel>.npz
                   the same run with the initial parameters perturbed by <rel>
                   relative: the reference's own sensitivity envelope
                   (``sens <rel>``; 1e-15 for the FP64 build, 1e-7 for FP32).
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

from qpinn.network import ModelConfig, build_model  # noqa: E402
from qpinn.physics import (CollocationGrid, LossEvaluator, MaterialMap,  # noqa: E402
                           time_bin_weights)
from qpinn.training import (AdamState, TrainConfig, adam_step, init_quantum_params,  # noqa: E402
                            lr_at, train)

HERE = os.path.dirname(os.path.abspath(__file__))
VAC = dict(variant="hybrid", ansatz="strongly", scale="acos", seed=0)


def step_headline(epochs=3, grid_dims=(64, 64, 16), t_end=1.5):
    """training.py:322-407 without the probes, one epoch at a time."""
    model = build_model(ModelConfig(**VAC, t_domain=t_end))
    params = model.init_params()
    params.quantum[:] = init_quantum_params("reg", model.n_quantum, 0)
    flat0 = params.flat.copy()
    grid = CollocationGrid(*grid_dims, t_end)
    ev = LossEvaluator(model, grid, MaterialMap("vacuum"), case="vacuum", energy_enabled=True,
                       chunk_slices=4)
    t0 = time.time()
    weights = time_bin_weights(ev.initial_bin_losses(params), 1.0)
    adam = AdamState.zeros(model.total_parameter_count)
    out = {k: [] for k in ("grad", "breakdown", "bin_phys", "weights", "flat")}
    for epoch in range(epochs):
        out["flat"].append(params.flat.copy())
        res = ev.evaluate(params, weights=weights, tape=True)
        bd = res.breakdown
        out["grad"].append(res.grad.copy())
        out["breakdown"].append([bd.phys, bd.ic, bd.sym, bd.energy, bd.total])
        out["bin_phys"].append(list(bd.bin_phys))
        out["weights"].append(weights.copy())
        adam_step(params, res.grad, adam, lr_at(epoch))
        weights = time_bin_weights(bd.bin_phys, 1.0)
        print(f"  epoch {epoch}: total {bd.total:.12e} ({time.time() - t0:.1f}s)", flush=True)
    s = grid.slice_size
    x, y, t = grid.flat_points()
    fields, derivs = model.forward(model.bind(ParamsAt(model, flat0)), x[:2 * s], y[:2 * s],
                                   t[:2 * s], derivs=True)
    np.savez_compressed(
        os.path.join(HERE, "step_headline.npz"),
        flat0=flat0, final_flat=params.flat, flat=np.array(out["flat"]),
        grad=np.array(out["grad"]),
        breakdown=np.array(out["breakdown"]), bin_phys=np.array(out["bin_phys"]),
        weights=np.array(out["weights"]), grid=np.array(grid_dims), t_end=np.array(t_end),
        fields=np.stack([fields.ez, fields.hx, fields.hy]),
        derivs=np.stack([derivs.ez, derivs.hx, derivs.hy]), forward_points=np.array(2 * s))


def ParamsAt(model, flat):
    p = model.init_params()
    p.flat[:] = flat
    return p


def curve_config1_perturbed(rel, epochs=1000, seed=7):
    """The reference trainer on config 1 with its initial parameters perturbed
    by ``rel`` relative (iid +-1 signs): the envelope of the reference's own
    sensitivity, against which a re-implementation's curve is judged (the late
    Adam phase of this run has loss spikes, where the trajectory is chaotic)."""
    import qpinn.training as RT
    orig = RT.init_quantum_params

    def perturbed_build(cfg):
        m = build_model(cfg)
        init = m.init_params

        def init_params():
            p = init()
            rng = np.random.default_rng(seed)
            p.flat[:m.n_classical] *= 1.0 + rel * rng.choice([-1.0, 1.0], m.n_classical)
            return p
        m.init_params = init_params
        return m

    def pq(strategy, count, s=0):
        q = orig(strategy, count, s)
        return q * (1.0 + rel * np.random.default_rng(seed + 1).choice([-1.0, 1.0], count))
    saved = (RT.build_model, RT.init_quantum_params)
    RT.build_model, RT.init_quantum_params = perturbed_build, pq
    try:
        rows = []
        tc = TrainConfig(case="vacuum", model=ModelConfig(**VAC), epochs=epochs, grid=(8, 8, 8),
                         energy_loss_enabled=True, eval_cadence=0, probe_cadence=0)
        train(tc, on_epoch=rows.append)
    finally:
        RT.build_model, RT.init_quantum_params = saved
    return np.array([r.total for r in rows])


def curve_config1(epochs=1000):
    """SURVEY 8(d) config 1 (pkg/configs/vacuum_qpinn.json model, 8x8x8 grid)."""
    rows = []
    tc = TrainConfig(case="vacuum", model=ModelConfig(**VAC), epochs=epochs, grid=(8, 8, 8),
                     energy_loss_enabled=True, eval_cadence=0, probe_cadence=0)
    t0 = time.time()
    res = train(tc, on_epoch=rows.append)
    print(f"  config1: {epochs} epochs in {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(
        os.path.join(HERE, "train_config1.npz"),
        total=np.array([r.total for r in rows]), phys=np.array([r.phys for r in rows]),
        ic=np.array([r.ic for r in rows]), sym=np.array([r.sym for r in rows]),
        energy=np.array([r.energy for r in rows]),
        bin_phys=np.array([r.bin_phys for r in rows]),
        grad_norm=np.array([r.grad_norm_all for r in rows]),
        final_flat=res.params.flat, grid=np.array((8, 8, 8)))


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("step", "all"):
        step_headline()
    if what in ("curve", "all"):
        curve_config1()
    if what in ("sens", "all"):
        rel = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-15
        tot = curve_config1_perturbed(rel)
        np.savez_compressed(os.path.join(HERE, f"train_config1_sens_{rel:.0e}.npz"), total=tot,
                            rel=np.array(rel))
