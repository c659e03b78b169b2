"""Known-answer and identity tests of the numpy oracle (CPU), after the reference's
own test strategy: gate algebra (test_qsim.py:41-59), <Z> = cos(theta)
(test_qsim.py:115-119), the acos / asin encoding identities (test_ansatz.py:135-146),
norm preservation (test_qsim.py:73-91), parameter-shift rules against the adjoint
gradient (test_qsim.py:139-166) and tangents against central differences
(test_autodiff.py:129-150).  These pin the oracle's arithmetic independently of the
golden vectors in test_oracle.py."""
import numpy as np
import pytest

from oracle import qpinn_oracle as O


def npar(kind, n, L):
    return O.build_circuit(kind, n, L)[1]


def test_gate_algebra():
    ket0 = np.array([1, 0], dtype=complex)
    assert np.allclose(O._rx(np.pi) @ ket0, [0, -1j], atol=1e-15)          # RX(pi)|0> = -i|1>
    assert np.allclose(O.u1_matrix("rot", [0.0, 0.0, 0.0]), np.eye(2), atol=1e-15)
    perm = O.permutation_for_cnots([(0, 1)], 2)                            # CNOT(0 -> 1)
    ket10 = np.zeros(4, dtype=complex)
    ket10[0b10] = 1.0
    assert np.argmax(np.abs(ket10[perm])) == 0b11                           # CNOT|10> = |11>
    for kind, th in (("rot", [0.3, -1.1, 2.0]), ("rxrz", [0.7, -0.4]), ("ry", [1.3])):
        U = O.u1_matrix(kind, th)
        assert np.allclose(U.conj().T @ U, np.eye(2), atol=1e-14)           # unitary


def test_expectation_z_is_cos_theta():
    rng = np.random.default_rng(1)
    a = rng.uniform(-1.0, 1.0, (64, 1))  # the domain rule holds for every scale
    qp = np.zeros(npar("no_entanglement", 1, 1))
    for scale, theta in (("none", a), ("pi", np.pi * a)):
        z, _ = O.pqc_forward(a, None, qp, "no_entanglement", scale, 1)
        assert np.max(np.abs(z - np.cos(theta))) <= 1e-12


@pytest.mark.parametrize("scale,sign", [("acos", 1.0), ("asin", -1.0)])
def test_encoding_identities(scale, sign):
    rng = np.random.default_rng(2)
    n, L = 7, 4
    a = rng.uniform(-0.99, 0.99, (32, n))
    qp = np.zeros(npar("no_entanglement", n, L))
    z, _ = O.pqc_forward(a, None, qp, "no_entanglement", scale, L)
    assert np.max(np.abs(z - sign * a)) <= 1e-10


@pytest.mark.parametrize("kind", ["strongly", "basic", "cross_mesh", "cross_mesh_2rot"])
def test_state_norm_preserved(kind):
    rng = np.random.default_rng(3)
    n, L = 6, 4
    a = rng.uniform(-0.9, 0.9, (16, n))
    qp = rng.uniform(0.0, 2 * np.pi, npar(kind, n, L))
    psi = O.pqc_state(a, qp, kind, "acos", L)
    assert np.max(np.abs(np.sum(np.abs(psi) ** 2, axis=-1) - 1.0)) <= 1e-10


def test_parameter_shift_matches_adjoint():
    """Every strongly-entangling slot sits in a single-axis rotation, so the
    two-term shift rule is exact for d(sum z)/d(theta)."""
    rng = np.random.default_rng(4)
    n, L, R = 4, 2, 8
    a = rng.uniform(-0.9, 0.9, (R, n))
    qp = rng.uniform(0.0, 2 * np.pi, npar("strongly", n, L))
    gz = np.ones((R, n))
    zeros = np.zeros((3, R, n))
    _, _, gq = O.pqc_backward(a, zeros, qp, "strongly", "acos", L, gz, zeros)

    def f(q):
        return O.pqc_forward(a, None, q, "strongly", "acos", L)[0].sum()

    shift = np.array([(f(qp + np.pi / 2 * e) - f(qp - np.pi / 2 * e)) / 2.0
                      for e in np.eye(qp.size)])
    assert np.max(np.abs(shift - gq)) <= 1e-10


def test_tangents_match_central_differences():
    rng = np.random.default_rng(5)
    n, L, R = 5, 3, 6
    a = rng.uniform(-0.8, 0.8, (R, n))
    da = rng.normal(size=(3, R, n))
    qp = rng.uniform(0.0, 2 * np.pi, npar("cross_mesh", n, L))
    _, dz = O.pqc_forward(a, da, qp, "cross_mesh", "asin", L)
    h = 1e-6
    for k in range(3):
        zp, _ = O.pqc_forward(a + h * da[k], None, qp, "cross_mesh", "asin", L)
        zm, _ = O.pqc_forward(a - h * da[k], None, qp, "cross_mesh", "asin", L)
        assert np.max(np.abs((zp - zm) / (2 * h) - dz[k])) <= 1e-7
