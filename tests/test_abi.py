"""C-ABI library: loads, exports every declared symbol, host-side circuit logic
(no GPU needed: the device plan upload is lazy)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
from conftest import ROOT, golden_cases

HEADER = os.path.join(ROOT, "include", "qpinn_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(qpinn_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2506_23246_b200 import _native as N
    lib = N.lib()
    names = _declared()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert {s[0] for s in N.SIGNATURES} == set(names)


def test_circuit_dump_matches_reference_for_every_ansatz():
    from paper_2506_23246_b200 import build_circuit
    for key, d in golden_cases("pqc_small.npz").items():
        kind = key.split("/")[0]
        c = build_circuit(kind, 3, 2)
        assert c.dump() == str(d["dump"])


@pytest.mark.parametrize("kind", O.KINDS)
@pytest.mark.parametrize("n,L", [(3, 2), (7, 4), (5, 7)])
def test_fused_plan_matches_oracle(kind, n, L):
    from paper_2506_23246_b200 import build_circuit
    c = build_circuit(kind, n, L)
    gates, P = O.build_circuit(kind, n, L)
    assert c.param_count == P
    want = O.fused_plan(gates, n)
    got = c.fused_plan()
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g[0] == w[0]
        if g[0] == "u1":
            assert (g[1], g[2], tuple(g[3])) == (w[1], w[2], tuple(int(s) for s in w[3]))
        elif g[0] == "perm":
            assert np.array_equal(np.asarray(g[1]), w[1])
        else:
            pm = O.crz_mesh_phase_matrix([(c_, t_) for c_, t_, _ in g[1]], n)
            assert np.array_equal(pm, w[1])
            assert [s for _, _, s in g[1]] == list(w[2])


def test_table1_param_counts():
    from paper_2506_23246_b200 import ansatz_param_count
    want = {"basic": 84, "strongly": 84, "cross_mesh": 196, "cross_mesh_2rot": 224,
            "cross_mesh_cnot": 84, "no_entanglement": 84}
    for k, v in want.items():
        assert ansatz_param_count(k, 7, 4) == v


def test_config_errors():
    from paper_2506_23246_b200 import ConfigError, build_circuit
    with pytest.raises(ConfigError):
        build_circuit("basic", 1, 1)
    with pytest.raises(ConfigError):
        build_circuit("strongly", 3, 0)
    with pytest.raises(ConfigError):
        build_circuit("nope", 3, 1)
    assert build_circuit("no_entanglement", 1, 1).param_count == 3


def test_quantum_layer_rejects_cpu_tensors():
    import torch
    from paper_2506_23246_b200 import ConfigError, quantum_layer_forward
    with pytest.raises(ConfigError):
        quantum_layer_forward(torch.zeros(4, 3, dtype=torch.float64), np.zeros(12), "strongly",
                              "acos")


@pytest.mark.parametrize("n,L,kind,fwd,bwd", [
    (4, 2, "strongly", "layer", "layer"),
    (7, 4, "strongly", "transfer", "transfer"),
    (8, 4, "cross_mesh", "transfer", "transfer"),
    (9, 1, "strongly", "cta/cluster", "cta/cluster"),
    (9, 4, "strongly", "transfer", "transfer"),
    (10, 8, "no_entanglement", "transfer", "transfer"),
    (11, 4, "strongly", "cta/cluster", "multi-gate HBM"),
    (11, 4, "cross_mesh", "cta/cluster", "cta/cluster"),
    (12, 1, "strongly", "cta/cluster", "multi-gate HBM"),
    (12, 4, "strongly", "multi-gate HBM", "multi-gate HBM"),
    (12, 4, "cross_mesh", "cta/cluster", "multi-gate HBM"),
    (13, 4, "cross_mesh", "multi-gate HBM", "multi-gate HBM"),
    (16, 8, "strongly", "multi-gate HBM", "multi-gate HBM"),
])
def test_float32_dispatch_table(n, L, kind, fwd, bwd):
    """The float32 K1 / K2 kernel choice (qpinn_pqc_regime) follows the measured
    dispatch table of DESIGN 3.1a / 3.3 (host-side logic, no GPU needed)."""
    import torch
    from paper_2506_23246_b200.ansatz import build_circuit
    c = build_circuit(kind, n, L)
    assert c.regime(torch.float32) == fwd
    assert c.regime(torch.float32, backward=True) == bwd
