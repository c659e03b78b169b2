"""Pin the numpy oracle to golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

import oracle as O
from conftest import golden_cases, load_golden


def _parse(key):
    parts = key.split("/")
    return parts


@pytest.mark.parametrize("fixture", ["pqc_small.npz", "pqc_n7.npz", "pqc_mid.npz"])
def test_oracle_pqc_matches_reference(fixture):
    worst = 0.0
    for key, d in golden_cases(fixture).items():
        parts = key.split("/")
        kind = parts[0]
        n = d["a"].shape[1]
        if fixture == "pqc_mid.npz":
            scale, L = "bias", int(parts[2])
        else:
            scale, L = parts[1], (2 if fixture == "pqc_small.npz" else 4)
        z, dz = O.pqc_forward(d["a"], d["da"], d["qp"], kind, scale, L)
        ga, gda, gq = O.pqc_backward(d["a"], d["da"], d["qp"], kind, scale, L, d["gz"], d["gdz"])
        zp, _ = O.pqc_forward(d["a"], None, d["qp"], kind, scale, L)
        for got, want in ((z, d["z"]), (dz, d["dz"]), (ga, d["ga"]), (gda, d["gda"]),
                          (gq, d["gq"]), (zp, d["zplain"])):
            err = np.max(np.abs(got - want)) / max(1.0, np.max(np.abs(want)))
            worst = max(worst, err)
    assert worst <= 1e-10, worst


def test_oracle_circuit_dump_matches_reference():
    for key, d in golden_cases("pqc_small.npz").items():
        kind = key.split("/")[0]
        gates, _ = O.build_circuit(kind, 3, 2)
        lines = []
        for k, w, s, src in gates:
            slots = "-" if not s else ("embed" if src == "embed" else "p") + ":" + ",".join(map(str, s))
            lines.append(f"{k} {','.join(map(str, w))} {slots}")
        assert "\n".join(lines) == str(d["dump"])


@pytest.mark.parametrize("name", ["eval_micro_vacuum.npz", "eval_micro_diel.npz",
                                  "eval_micro_asym.npz", "eval_desk.npz",
                                  "eval_vacuum7.npz", "eval_diel7.npz",
                                  "eval_n6_strongly.npz", "eval_n6_crossmesh.npz",
                                  "eval_n8_strongly.npz", "eval_n9_crossmesh.npz",
                                  "eval_n10_2rot.npz", "eval_n12_strongly.npz"])
def test_oracle_evaluate_matches_reference(name):
    g = load_golden(name)
    h, F, n, L, seed = (int(v) for v in g["config"])
    t_end = float(g["t_end"])
    model = O.OracleModel(hidden=h, rff=F, n_qubits=n, n_layers=L, ansatz=str(g["ansatz"]),
                          scale=str(g["scale"]), seed=seed, t_domain=float(g["t_domain"]))
    flat = model.init_params()
    assert np.array_equal(flat, g["flat"])
    grid = O.Grid(*(int(v) for v in g["grid"]), t_end)
    ev = O.Evaluator(model, grid, case=str(g["case"]), phys_mode=str(g["phys_mode"]),
                     energy=bool(g["energy"]), chunk_slices=int(g["chunk_slices"]))
    w = g["weights"] if g["weights"].size else None
    bd, grad, _ = ev.evaluate(flat, w, tape=True)
    want = g["breakdown"]
    got = np.array([bd[k] for k in ("phys", "ic", "sym", "energy", "total")])
    assert np.allclose(got, want, rtol=1e-11, atol=1e-14)
    assert np.allclose(bd["bin_phys"], g["bin_phys"], rtol=1e-11, atol=1e-14)
    assert np.max(np.abs(grad - g["grad"])) <= 1e-10 * max(1.0, np.max(np.abs(g["grad"])))
    out, dout, _ = model.forward(flat, *(np.concatenate([a] * 1) for a in (
        np.tile(grid.x_slice, grid.nt), np.tile(grid.y_slice, grid.nt),
        np.repeat(grid.ts, grid.s))))
    assert np.allclose(out.T, g["fields"], rtol=1e-11, atol=1e-13)
    assert np.allclose(np.transpose(dout, (2, 0, 1)), g["derivs"], rtol=1e-10, atol=1e-12)


def test_oracle_train_curve_matches_reference_desk():
    g = load_golden("train_desk.npz")
    h, F, n, L, seed = (int(v) for v in g["config"])
    model = O.OracleModel(hidden=h, rff=F, n_qubits=n, n_layers=L, ansatz=str(g["ansatz"]),
                          scale=str(g["scale"]), seed=seed, t_domain=1.5)
    epochs = 60
    rows, flat = O.train_curve(model, O.Grid(*(int(v) for v in g["grid"]), 1.5), epochs)
    tot = np.array([r["total"] for r in rows])
    rel = np.max(np.abs(tot - g["total"][:epochs]) / np.abs(g["total"][:epochs]))
    assert rel <= 1e-9, rel


def test_oracle_shard_sum_is_exact():
    """Sharding whole time slices and summing reproduces the full gradient."""
    g = load_golden("eval_micro_vacuum.npz")
    model = O.OracleModel(hidden=6, rff=5, n_qubits=3, n_layers=2, ansatz="strongly",
                          scale="acos", seed=3)
    flat = model.init_params()
    grid = O.Grid(4, 4, 7, 1.5)
    w = g["weights"]
    full = O.Evaluator(model, grid, chunk_slices=2).evaluate(flat, w, tape=True)
    parts = [O.Evaluator(model, grid, chunk_slices=2, slices=s).evaluate(flat, w, tape=True)
             for s in ([0, 1, 2], [3, 4], [5, 6])]
    gsum = sum(p[1] for p in parts)
    assert np.max(np.abs(gsum - full[1])) <= 1e-13 * np.max(np.abs(full[1]))
