"""GPU FDTD solver (qpinn_fdtd_run) against the reference's own snapshots
(tests/golden/fdtd_*.npz, fdtd.py:115-181).  Every update is rounded in the
reference's order; the initial exp/cos may differ from numpy's by an ulp, so
the bar is 1e-13 relative to the field scale (measured: see the assertion
messages), and the plane wave additionally checks the scheme's known
second-order accuracy against the exact solution."""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _cfg(g):
    from paper_2506_23246_b200.fdtd import FdtdConfig
    nx, ny, ns = (int(v) for v in g["config"])
    return FdtdConfig(nx=nx, ny=ny, case=str(g["case"]), t_end=float(g["t_end"]),
                      cfl=float(g["cfl"]), ic=str(g["ic"]), n_snapshots=ns,
                      eps_r=float(g["eps_r"]), slab_x0=float(g["slab_x0"]))


@pytest.mark.parametrize("name", ["fdtd_vacuum.npz", "fdtd_dielectric.npz", "fdtd_plane.npz"])
def test_fdtd_matches_reference(name):
    from paper_2506_23246_b200.fdtd import energy_history, run_reference
    g = load_golden(name)
    h = run_reference(_cfg(g))
    assert h.meta["steps"] == int(g["steps"]) and h.meta["dt"] == float(g["dt"])
    assert np.array_equal(h.times, g["times"])
    assert np.array_equal(h.xs, g["xs"]) and np.array_equal(h.ys, g["ys"])
    for k in ("ez", "hx", "hy"):
        got, want = getattr(h, k), g[k]
        err = np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300)
        assert err <= 1e-13, (k, err)
    assert np.allclose(energy_history(h), g["energy"], rtol=1e-13)


def test_fdtd_save_load_roundtrip(tmp_path):
    from paper_2506_23246_b200.fdtd import FdtdConfig, FieldHistory, run_reference
    h = run_reference(FdtdConfig(nx=16, ny=12, n_snapshots=3))
    h.save(str(tmp_path))
    h2 = FieldHistory.load(str(tmp_path))
    for k in ("ez", "hx", "hy", "times", "xs", "ys"):
        assert np.array_equal(getattr(h, k), getattr(h2, k))


def test_fdtd_plane_wave_second_order():
    """Ez = cos(pi (x + t)) is exact; the max error falls ~4x per grid halving."""
    from paper_2506_23246_b200.fdtd import FdtdConfig, run_reference
    errs = []
    for nx in (32, 64, 128):
        h = run_reference(FdtdConfig(nx=nx, ny=4, ic="plane_wave", t_end=0.5, n_snapshots=2))
        exact = np.cos(np.pi * (h.xs[None, :] + h.times[-1]))
        errs.append(np.max(np.abs(h.ez[-1] - exact)))
    assert errs[0] / errs[1] > 3.5 and errs[1] / errs[2] > 3.5, errs
