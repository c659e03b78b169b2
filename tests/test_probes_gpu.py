"""Diagnostic probes on the native inference engine against
the reference's golden vectors (tests/golden/make_golden_probes.py):
value-only predict, Meyer-Wallach Q, energy probe + black-hole index, L2 vs
an FDTD history.  float64: 1e-10 relative; float32: 2e-5 relative (value
path through the 3xTF32 tensor-core trunk and the fp32 circuit)."""
import numpy as np
import pytest
import torch

from conftest import load_golden

pytestmark = pytest.mark.gpu

TOL = {torch.float64: 1e-10, torch.float32: 2e-5}


def _model(g, dtype):
    from paper_2506_23246_b200.network import ModelConfig, build_model
    h, F, n, L, seed = (int(v) for v in g["config"])
    cfg = ModelConfig(variant="hybrid", hidden_width=h, rff_features=F, n_qubits=n,
                      n_layers_pqc=L, ansatz=str(g["ansatz"]), scale=str(g["scale"]), seed=seed,
                      t_domain=float(g["t_domain"]))
    return build_model(cfg, device="cuda", dtype=dtype)


def _rel(got, want):
    got, want = np.asarray(got, float), np.asarray(want, float)
    return float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300))


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("name", ["probes_desk.npz", "probes_vacuum7.npz"])
def test_probes_match_reference(name, dtype):
    from paper_2506_23246_b200.fdtd import FieldHistory
    from paper_2506_23246_b200.physics import MaterialMap
    from paper_2506_23246_b200.probes import (bh_index, energy_probe, l2_against_reference,
                                              probe_entanglement)
    g = load_golden(name)
    m = _model(g, dtype)
    params = m.init_params()
    assert np.array_equal(params.flat.double().cpu().numpy(), g["flat"].astype(
        np.float32 if dtype == torch.float32 else np.float64).astype(np.float64))
    tol = TOL[dtype]
    fb = m.predict(params, g["px"], g["py"], g["pt"])
    pred = np.stack([v.double().cpu().numpy() for v in (fb.ez, fb.hx, fb.hy)])
    assert _rel(pred, g["pred"]) <= tol
    mw = probe_entanglement(m, params, g["mw_x"], g["mw_y"], g["mw_t"])
    assert abs(mw - float(g["mw"])) <= tol * abs(float(g["mw"]))
    nx, ny, nt = (int(v) for v in g["probe_grid"])
    u = energy_probe(m, params, MaterialMap(case=str(g["case"])), nx, ny, g["times"])
    assert _rel(u, g["energy"]) <= tol
    ib = bh_index(u, g["times"])
    assert abs(ib[1] - float(g["i_bh"][1])) <= 10 * tol
    f = load_golden("fdtd_vacuum.npz")
    hist = FieldHistory(times=f["times"], ez=f["ez"], hx=f["hx"], hy=f["hy"], xs=f["xs"],
                        ys=f["ys"])
    l2 = l2_against_reference(m, params, hist)
    assert abs(l2 - float(g["l2"])) <= tol * abs(float(g["l2"]))


def test_predict_native_matches_autograd_path():
    """The native value path equals the autograd forward (torch trunk) in fp64."""
    from paper_2506_23246_b200.network import ModelConfig, build_model
    m = build_model(ModelConfig(variant="hybrid", ansatz="cross_mesh_2rot", scale="bias",
                                seed=4), device="cuda", dtype=torch.float64)
    p = m.init_params()
    rng = np.random.default_rng(3)
    x, y, t = rng.uniform(-1, 1, 777), rng.uniform(-1, 1, 777), rng.uniform(0, 1.5, 777)
    fb = m.predict(p, x, y, t)
    ref, _ = m.forward(p, x, y, t, native=False)
    for a, b in zip((fb.ez, fb.hx, fb.hy), (ref.ez, ref.hx, ref.hy)):
        assert torch.allclose(a, b, rtol=1e-11, atol=1e-12)
    # Model.forward itself (native by default) with and without jacobians
    nat, dnat = m.forward(p, x, y, t, derivs=True)
    ref, dref = m.forward(p, x, y, t, derivs=True, native=False)
    for a, b in zip((nat.ez, nat.hx, nat.hy, dnat.ez, dnat.hx, dnat.hy),
                    (ref.ez, ref.hx, ref.hy, dref.ez, dref.hx, dref.hy)):
        assert torch.allclose(a, b, rtol=1e-11, atol=1e-12)
    a_nat = m.adapter_activations(p, x, y, t)
    pv = m.views(p.flat)
    X, Y, T = m._coords(x, y, t)
    h, _ = m.trunk(pv, X, Y, T, False)
    assert torch.allclose(a_nat, torch.tanh(h @ pv["adapter.W"] + pv["adapter.b"]),
                          rtol=1e-11, atol=1e-12)


def test_train_with_probes_matches_reference():
    """train() with every probe on (training.py:365-391), float64: loss curve,
    per-epoch Meyer-Wallach Q, black-hole index and L2 columns."""
    from paper_2506_23246_b200.fdtd import FieldHistory
    from paper_2506_23246_b200.network import ModelConfig
    from paper_2506_23246_b200.training import TrainConfig, train
    g = load_golden("train_probes_desk.npz")
    f = load_golden("fdtd_vacuum.npz")
    hist = FieldHistory(times=f["times"], ez=f["ez"], hx=f["hx"], hy=f["hy"], xs=f["xs"],
                        ys=f["ys"])
    h, F, n, L, seed = (int(v) for v in g["config"])
    cfg = TrainConfig(case="vacuum", model=ModelConfig(variant="hybrid", hidden_width=h,
                      rff_features=F, n_qubits=n, n_layers_pqc=L, ansatz=str(g["ansatz"]),
                      scale=str(g["scale"]), seed=seed), epochs=int(g["epochs"]),
                      grid=(8, 8, 10), eval_cadence=10, probe_cadence=10, probe_grid=(8, 8, 6))
    res = train(cfg, reference=hist, dtype=torch.float64)
    rows = res.log.rows
    assert _rel([r.total for r in rows], g["total"]) <= 1e-9
    assert _rel([r.mw_q for r in rows], g["mw"]) <= 1e-9
    for key, col in (("i_bh", g["i_bh"]), ("l2_err", g["l2"])):
        got = np.array([np.nan if getattr(r, key) is None else getattr(r, key) for r in rows])
        assert np.array_equal(np.isnan(got), np.isnan(col)), key
        ok = ~np.isnan(col)
        assert _rel(got[ok], col[ok]) <= 1e-8, key
    assert abs(res.log.final_l2 - float(g["final_l2"])) <= 1e-8 * float(g["final_l2"])
    assert _rel(res.log.energy_history, g["energy_history"]) <= 1e-8
