"""Generate golden vectors from the reference implementation itself.

Run in the build container (the reference is importable only here):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``qpinn`` from /root/reference/pkg/src (read-only) and writes small
``.npz`` fixtures next to this script.  The GPU box never reads
/root/reference; it only reads these committed files.

Fixtures
--------
pqc_small.npz     quantum_layer_forward (ansatz.py:341-400) values + tangents and
                  taped gradients (tape.py:118-148) for every ansatz x scale at n=3,L=2
pqc_n7.npz        same for every ansatz at the default 7 qubits x 4 layers (acos/asin)
pqc_mid.npz       n=4..6 at several layer counts (strongly/cross_mesh, bias)
eval_*.npz        LossEvaluator.evaluate(tape=True) breakdown + full flat gradient
                  (physics.py:334-428) on small grids for several model configs
train_*.npz       per-epoch loss curves of training.train (training.py:309-414)
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

from qpinn import ansatz as RA  # noqa: E402
from qpinn.autodiff.ops import BatchedDual  # noqa: E402
from qpinn.autodiff.tape import Tensor  # noqa: E402
from qpinn.network import ModelConfig, build_model  # noqa: E402
from qpinn.physics import (CollocationGrid, LossEvaluator, MaterialMap,  # noqa: E402
                           time_bin_weights)
from qpinn.training import TrainConfig, train  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
KINDS = [k.value for k in RA.AnsatzKind]
SCALES = [s.value for s in RA.ScaleKind]


def pqc_case(rng, kind, scale, n, L, R, amax=0.9):
    circ = RA.build_circuit(kind, n, L)
    qp = rng.uniform(0, 2 * np.pi, circ.param_count)
    a = rng.uniform(-amax, amax, (R, n))
    da = rng.normal(size=(3, R, n))
    gz = rng.normal(size=(R, n))
    gdz = rng.normal(size=(3, R, n))
    av, at, qt = Tensor(a), Tensor(da), Tensor(qp)
    B = RA._ansatz_transfer(circ, qt)
    out = RA.quantum_layer_forward(BatchedDual(av, at), qt, circ, scale, transfer=B)
    loss = (out.val * gz).sum() + (out.tan * gdz).sum()
    loss.backward()
    zplain = RA.quantum_layer_forward(a, qp, circ, scale)
    return dict(a=a, da=da, qp=qp, gz=gz, gdz=gdz, z=out.val.value, dz=out.tan.value,
                ga=av.grad, gda=at.grad, gq=qt.grad, zplain=zplain,
                dump=np.array(circ.dump()))


def save_pqc(name, cases):
    flat = {}
    for key, d in cases.items():
        for k, v in d.items():
            flat[f"{key}/{k}"] = v
    np.savez_compressed(os.path.join(HERE, name), **flat)


def eval_case(name, cfg, grid_dims, case, t_end=1.5, chunk_slices=2, weights=None,
              energy=True, phys_mode=None):
    model = build_model(cfg)
    params = model.init_params()
    grid = CollocationGrid(*grid_dims, t_end)
    ev = LossEvaluator(model, grid, MaterialMap(case), case=case, phys_mode=phys_mode,
                       energy_enabled=energy, chunk_slices=chunk_slices)
    res = ev.evaluate(params, weights=weights, tape=True)
    bd = res.breakdown
    plain = ev.evaluate(params, weights=weights).breakdown
    x, y, t = grid.flat_points()
    fields, derivs = model.forward(model.bind(params), x, y, t, derivs=True)
    np.savez_compressed(
        os.path.join(HERE, name),
        flat=params.flat, grad=res.grad,
        weights=np.asarray(weights if weights is not None else []),
        breakdown=np.array([bd.phys, bd.ic, bd.sym, bd.energy, bd.total]),
        bin_phys=np.array(bd.bin_phys), plain_total=np.array(plain.total),
        fields=np.stack([fields.ez, fields.hx, fields.hy]),
        derivs=np.stack([derivs.ez, derivs.hx, derivs.hy]),
        grid=np.array(grid_dims), t_end=np.array(t_end), case=np.array(case),
        energy=np.array(energy), chunk_slices=np.array(chunk_slices),
        phys_mode=np.array(ev.phys_mode),
        config=np.array([cfg.hidden_width, cfg.rff_features, cfg.n_qubits,
                         cfg.n_layers_pqc, cfg.seed]),
        t_domain=np.array(cfg.t_domain),
        ansatz=np.array(cfg.ansatz), scale=np.array(cfg.scale))


def train_case(name, cfg_model, grid, epochs, case="vacuum", energy=True):
    rows = []
    tc = TrainConfig(case=case, model=cfg_model, epochs=epochs, grid=grid,
                     energy_loss_enabled=energy, eval_cadence=0, probe_cadence=0)
    t0 = time.time()
    res = train(tc, on_epoch=rows.append)
    print(f"  {name}: {epochs} epochs in {time.time() - t0:.1f}s")
    np.savez_compressed(
        os.path.join(HERE, name),
        total=np.array([r.total for r in rows]), phys=np.array([r.phys for r in rows]),
        ic=np.array([r.ic for r in rows]), sym=np.array([r.sym for r in rows]),
        energy=np.array([r.energy for r in rows]),
        bin_phys=np.array([r.bin_phys for r in rows]),
        grad_norm=np.array([r.grad_norm_all for r in rows]),
        final_flat=res.params.flat, grid=np.array(grid), case=np.array(case),
        energy_enabled=np.array(energy),
        config=np.array([cfg_model.hidden_width, cfg_model.rff_features,
                         cfg_model.n_qubits, cfg_model.n_layers_pqc, cfg_model.seed]),
        ansatz=np.array(cfg_model.ansatz), scale=np.array(cfg_model.scale))


def main():
    rng = np.random.default_rng(20250623)
    cases = {f"{k}/{s}": pqc_case(rng, k, s, 3, 2, 6) for k in KINDS for s in SCALES}
    # near-singular acos/asin inputs (|a| up to 0.995) exercise S' and S''
    cases.update({f"{k}/{s}/edge": pqc_case(rng, k, s, 3, 2, 6, amax=0.995)
                  for k in ("strongly", "cross_mesh") for s in ("acos", "asin")})
    save_pqc("pqc_small.npz", cases)
    save_pqc("pqc_n7.npz", {f"{k}/{s}": pqc_case(rng, k, s, 7, 4, 12)
                            for k in KINDS for s in ("acos", "asin")})
    mid = {}
    for n in (4, 5, 6):
        for L in (1, 3, 5):
            for k in ("strongly", "cross_mesh", "cross_mesh_2rot"):
                mid[f"{k}/{n}/{L}"] = pqc_case(rng, k, "bias", n, L, 5)
    save_pqc("pqc_mid.npz", mid)

    micro = dict(variant="hybrid", hidden_width=6, rff_features=5, n_qubits=3,
                 n_layers_pqc=2, ansatz="strongly", scale="acos", seed=3, t_domain=1.5)
    w = np.array([1.0, 0.8, 0.5, 0.2, 0.05])
    eval_case("eval_micro_vacuum.npz", ModelConfig(**micro), (4, 4, 7), "vacuum",
              weights=w)
    eval_case("eval_micro_diel.npz", ModelConfig(**{**micro, "ansatz": "cross_mesh_2rot",
                                                    "scale": "asin"}),
              (6, 4, 5), "dielectric", t_end=0.7, weights=w, energy=False)
    eval_case("eval_micro_asym.npz", ModelConfig(**{**micro, "ansatz": "cross_mesh",
                                                    "scale": "pi"}),
              (4, 6, 6), "asymmetric", weights=None)
    desk = dict(variant="hybrid", hidden_width=16, rff_features=8, n_qubits=4,
                n_layers_pqc=2, ansatz="strongly", scale="acos", seed=0, t_domain=1.5)
    eval_case("eval_desk.npz", ModelConfig(**desk), (8, 8, 10), "vacuum", chunk_slices=4,
              weights=w)
    vac = dict(variant="hybrid", ansatz="strongly", scale="acos", seed=0, t_domain=1.5)
    eval_case("eval_vacuum7.npz", ModelConfig(**vac), (4, 4, 6), "vacuum", chunk_slices=4,
              weights=w)
    eval_case("eval_diel7.npz", ModelConfig(**{**vac, "ansatz": "no_entanglement",
                                                "scale": "asin", "t_domain": 0.7}),
              (6, 4, 5), "dielectric", t_end=0.7, chunk_slices=4, weights=w, energy=False)

    train_case("train_desk.npz", ModelConfig(**desk), (8, 8, 10), 1000)
    train_case("train_vacuum7.npz", ModelConfig(**vac), (4, 4, 6), 200)


if __name__ == "__main__":
    main()
