"""The oracle's probe and FDTD restatements against the reference's own
golden vectors (tests/golden/make_golden_probes.py): Meyer-Wallach Q, the
energy probe and black-hole index, value-only predictions, L2 vs FDTD, and
the Yee solver's snapshots.  CPU only."""
import numpy as np
import pytest

import oracle as O
from conftest import load_golden


def _model(g):
    h, F, n, L, seed = (int(v) for v in g["config"])
    return O.OracleModel(hidden=h, rff=F, n_qubits=n, n_layers=L, ansatz=str(g["ansatz"]),
                         scale=str(g["scale"]), seed=seed, t_domain=float(g["t_domain"]))


@pytest.mark.parametrize("name", ["probes_desk.npz", "probes_vacuum7.npz"])
def test_oracle_probes_match_reference(name):
    g = load_golden(name)
    m = _model(g)
    flat = m.init_params()
    assert np.array_equal(flat, g["flat"])
    mw = O.probe_entanglement(m, flat, g["mw_x"], g["mw_y"], g["mw_t"])
    assert abs(mw - float(g["mw"])) <= 1e-12
    pred = O.model_predict(m, flat, g["px"], g["py"], g["pt"])
    assert np.allclose(pred, g["pred"], rtol=1e-11, atol=1e-13)
    nx, ny, nt = (int(v) for v in g["probe_grid"])
    u = O.energy_probe(m, flat, str(g["case"]), nx, ny, g["times"])
    assert np.allclose(u, g["energy"], rtol=1e-12)
    assert np.allclose(O.bh_index(u, g["times"]), g["i_bh"], rtol=1e-10, atol=1e-13)
    f = load_golden("fdtd_vacuum.npz")
    l2 = O.l2_against_reference(m, flat, f["times"], f["xs"], f["ys"], f["ez"])
    assert abs(l2 - float(g["l2"])) <= 1e-11 * abs(float(g["l2"]))


@pytest.mark.parametrize("name", ["fdtd_vacuum.npz", "fdtd_dielectric.npz", "fdtd_plane.npz"])
def test_oracle_fdtd_matches_reference(name):
    g = load_golden(name)
    nx, ny, ns = (int(v) for v in g["config"])
    r = O.fdtd_run(nx, ny, case=str(g["case"]), t_end=float(g["t_end"]), cfl=float(g["cfl"]),
                   ic=str(g["ic"]), n_snapshots=ns, eps_r=float(g["eps_r"]),
                   slab_x0=float(g["slab_x0"]))
    assert r["steps"] == int(g["steps"]) and r["dt"] == float(g["dt"])
    assert np.array_equal(r["times"], g["times"])
    for k in ("ez", "hx", "hy"):
        assert np.array_equal(r[k], g[k]), k  # same numpy operations in the same order
    u = [O.total_energy(r["ez"][i], r["hx"][i], r["hy"][i], r["eps"], 2.0 / nx, 2.0 / ny)
         for i in range(len(r["times"]))]
    assert np.allclose(u, g["energy"], rtol=1e-13)


def test_oracle_meyer_wallach_known_states():
    # product state -> 0; GHZ -> 1; |+>|0> product -> 0
    n = 3
    prod = np.zeros(8, complex)
    prod[0] = 1.0
    ghz = np.zeros(8, complex)
    ghz[0] = ghz[7] = 2 ** -0.5
    assert abs(O.meyer_wallach(prod)[0]) < 1e-15
    assert abs(O.meyer_wallach(ghz)[0] - 1.0) < 1e-15
    assert O.meyer_wallach(np.ones((2, 8)) / np.sqrt(8)).shape == (2,)
    del n
