"""The reference package itself, patched onto the C ABI through the ctypes stub
of INTEGRATION.md §2 (``tests/ref_binding.py``), reproduces its own unpatched
``LossEvaluator.evaluate(tape=True)`` (the golden vectors the unpatched
reference wrote) -- the drop-in claim of SURVEY §8(b), end to end.

The installed reference (``baseline/_ref``, pure Python) travels to the GPU box
with the repository snapshot; ``/root/reference`` is never read here."""
import os
import sys

import numpy as np
import pytest
import torch

from conftest import ROOT, load_golden
from gpu_util import assert_close

REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(ROOT, "tests")


def _qpinn():
    if not os.path.isdir(os.path.join(REF, "qpinn")):
        pytest.skip("baseline/_ref (the installed reference) is absent")
    for p in (REF, TESTS):
        if p not in sys.path:
            sys.path.insert(0, p)
    import qpinn
    return qpinn


def _reference_evaluator(g):
    from qpinn.network import ModelConfig, build_model
    from qpinn.physics import CollocationGrid, LossEvaluator, MaterialMap
    h, F, n, L, seed = (int(v) for v in g["config"])
    cfg = ModelConfig(variant="hybrid", hidden_width=h, rff_features=F, n_qubits=n,
                      n_layers_pqc=L, ansatz=str(g["ansatz"]), scale=str(g["scale"]), seed=seed,
                      t_domain=float(g["t_domain"]))
    model = build_model(cfg)
    grid = CollocationGrid(*(int(v) for v in g["grid"]), float(g["t_end"]))
    case = str(g["case"])
    ev = LossEvaluator(model, grid, MaterialMap(case), case=case, phys_mode=str(g["phys_mode"]),
                       energy_enabled=bool(g["energy"]), chunk_slices=int(g["chunk_slices"]))
    return model, grid, ev


def test_stub_argtypes_match_the_header():
    """The stub's ctypes arity equals the C declarations (the round-1 stub had
    12 argtypes for the 13-argument qpinn_pqc_forward)."""
    import re
    if TESTS not in sys.path:
        sys.path.insert(0, TESTS)
    import ref_binding
    with open(os.path.join(ROOT, "include", "qpinn_b200.h")) as f:
        hdr = f.read()

    class FakeFn:
        argtypes = None
        restype = None

    class FakeLib:
        def __getattr__(self, name):
            fn = FakeFn()
            object.__setattr__(self, name, fn)
            return fn
    lib = ref_binding._bind(FakeLib())
    for name in ("qpinn_pqc_forward", "qpinn_pqc_backward", "qpinn_pqc_workspace_bytes",
                 "qpinn_pqc_state_bytes", "qpinn_pqc_domain_check", "qpinn_circuit_create"):
        m = re.search(r"\b" + name + r"\s*\(([^;]*?)\)\s*;", hdr, re.S)
        assert m, name
        nargs = len([a for a in m.group(1).split(",") if a.strip()])
        assert len(getattr(lib, name).argtypes) == nargs, name
    assert lib.qpinn_last_error.restype is __import__("ctypes").c_char_p


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["eval_vacuum7.npz", "eval_desk.npz"])
def test_reference_evaluate_through_the_abi(name):
    qpinn = _qpinn()
    import ref_binding
    g = load_golden(name)
    uninstall = ref_binding.install(qpinn, torch.float64)
    try:
        model, grid, ev = _reference_evaluator(g)
        params = model.init_params()
        assert np.array_equal(params.flat, g["flat"])
        w = g["weights"] if g["weights"].size else None
        res = ev.evaluate(params, weights=w, tape=True)
        bd = res.breakdown
        got = np.array([bd.phys, bd.ic, bd.sym, bd.energy, bd.total])
        assert_close(got, g["breakdown"], torch.float64, "breakdown (reference through the ABI)")
        assert_close(np.array(bd.bin_phys), g["bin_phys"], torch.float64, "bin_phys")
        assert_close(res.grad, g["grad"], torch.float64, "flat gradient (reference through the ABI)")
        plain = ev.evaluate(params, weights=w, tape=False)
        assert abs(plain.breakdown.total - float(g["plain_total"])) <= 1e-10 * abs(
            float(g["plain_total"]))
        x, y, t = grid.flat_points()
        fields, derivs = model.forward(model.bind(params), x, y, t, derivs=True)
        assert_close(np.stack([fields.ez, fields.hx, fields.hy]), g["fields"], torch.float64,
                     "fields")
        assert_close(np.stack([derivs.ez, derivs.hx, derivs.hy]), g["derivs"], torch.float64,
                     "derivs")
    finally:
        uninstall()


@pytest.mark.gpu
def test_reference_domain_rule_through_the_abi():
    """DomainError / clamp warning of ansatz.py:51-58 come back through the stub."""
    qpinn = _qpinn()
    import ref_binding
    from qpinn.ansatz import build_circuit
    from qpinn.autodiff.ops import BatchedDual
    from qpinn.errors import DomainError
    qlf = ref_binding.make_quantum_layer_forward(torch.float64)
    circ = build_circuit("strongly", 4, 2)
    rng = np.random.default_rng(0)
    qp = rng.uniform(0, 2 * np.pi, circ.param_count)
    a = rng.uniform(-0.9, 0.9, (8, 4))
    da = rng.normal(size=(3, 8, 4))
    a[3, 1] = 1.0 + 1e-9
    with pytest.raises(DomainError):
        qlf(BatchedDual(a, da), qp, circ, "acos")
    a[3, 1] = 1.0 + 1e-13
    with pytest.warns(UserWarning, match="clamped"):
        qlf(BatchedDual(a, da), qp, circ, "acos")
    from qpinn.errors import ConfigError
    with pytest.raises(ConfigError):
        qlf(BatchedDual(a[:, :3], da[:, :, :3]), qp, circ, "acos")
