"""Algorithmic work per collocation point, derived from the fused plan.

Conventions: 8 FLOP per complex MAC; a dense 2x2 gate on one
state = D/2 pairs x 4 MACs = 16 D; a diagonal phase step = 6 D; a
permutation = 0; 4 states (psi and its x/y/t tangents).
  F_fwd+tan = 4 (16 D n_u1 + 6 D n_phase) + 32 D (embedding) + 4 D (n + 4) (readout)
  F_adjoint = 2 x the 4-state ansatz term (propagate 4 adjoints, 2x2
              outer-product accumulation per gate); the layer-boundary states
              K1 checkpoints mean no state is un-computed
For 7 qubits x 4 layers (strongly): 2.39e5 and 4.59e5 FLOP/point.
"""
from __future__ import annotations


def pqc_flops(circuit):
    n = circuit.n_qubits
    D = 1 << n
    plan = circuit.fused_plan()
    n_u1 = sum(1 for s in plan if s[0] == "u1")
    n_ph = sum(1 for s in plan if s[0] == "phases")
    ansatz = 16 * D * n_u1 + 6 * D * n_ph
    f_fwd = 4 * ansatz + 32 * D + 4 * D * (n + 4)
    f_adj = 2 * 4 * ansatz
    return f_fwd, f_adj


def trunk_flops(hidden: int = 128, rff: int = 128, n_qubits: int = 7, n_hidden: int = 3):
    """Trunk forward with tangents (4 channels) and backward (~2x), SURVEY 8d."""
    w_in = 2 * rff
    fwd = 2 * 4 * (6 * rff + w_in * hidden + (n_hidden - 1) * hidden * hidden
                   + hidden * n_qubits + n_qubits * 3)
    return fwd, 2 * fwd
