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


def transfer_bytes(n: int):
    """HBM bytes per point of the transfer-matrix K1/K2 (pqc_transfer.cu, float32).
    A [4 rows, 2D] operand (Psi, Abar) is 4 x 2D x 4 = 32 D bytes per point; the
    embedded magnitudes m and dL/dm (the phase lives in W', tr_wmat) are 16 D.
      forward : embed writes m (16 D); the GEMM reads m, writes Psi (16 D + 32 D)
                and reduces the readout in its epilogue (n = 7); a, da in and
                z, dz out (2 x 16 n)
      backward: seeds read Psi, write Abar (2 x 32 D); the GEMM reads Abar, writes
                dL/dm (32 D + 16 D); the embedding gradient reads dL/dm (16 D); the
                weight-gradient GEMM reads m and Abar (16 D + 32 D) + dL/dz, dL/ddz,
                a, da in, g_a, g_da out (3 x 16 n)
    The D x 2D transfer matrix and its adjoint are L2-resident and not counted."""
    D = 1 << n
    fwd = (64 if n == 7 else 96) * D  # n = 7: the readout is fused into the map's epilogue
    return fwd + 2 * 16 * n, 176 * D + 3 * 16 * n


def transfer_flops(n: int):
    """Algorithmic (fp32) GEMM flops per point: Psi = m W' is [4, D] x [D, 2D];
    the backward has dL/dm = Abar W'^T and dL/dW' += m^T Abar."""
    D = 1 << n
    return 2 * 4 * D * 2 * D, 2 * 2 * 4 * D * 2 * D


def trunk_flops(hidden: int = 128, rff: int = 128, n_qubits: int = 7, n_hidden: int = 3):
    """Trunk forward with tangents (4 channels) and backward (~2x), SURVEY 8d."""
    w_in = 2 * rff
    fwd = 2 * 4 * (6 * rff + w_in * hidden + (n_hidden - 1) * hidden * hidden
                   + hidden * n_qubits + n_qubits * 3)
    return fwd, 2 * fwd


def trunk_bytes(hidden: int = 128, rff: int = 128, n_qubits: int = 7, n_hidden: int = 3,
                elem: int = 4):
    """HBM bytes per point the trunk passes must move (4 channels of every
    activation; weights are L2-resident and not counted), per the fused
    kernels of trunk.cu / tc_gemm.cu:
      forward : features write H0, then every dense layer reads its input and
                writes its dual-tanh output once
      backward: per hidden layer the dual-tanh reverse (read dL/dH and H, write
                dL/dU), the weight gradient (read H_in, dL/dU), the input
                gradient (read dL/dU, write dL/dH_in) and the bias sum (read
                dL/dU value channel); adapter likewise; tau (read dL/dH0)."""
    c = 4 * elem
    widths = [2 * rff] + [hidden] * n_hidden + [n_qubits]
    fwd = 3 * elem + c * widths[0]
    for k, n in zip(widths[:-1], widths[1:]):
        fwd += c * (k + n)
    bwd = 0
    for k, n in zip(widths[:-1], widths[1:]):
        bwd += 3 * c * n          # tanh reverse
        bwd += c * (k + n)        # weight gradient
        bwd += c * (n + k)        # input gradient
        bwd += elem * n           # bias sum
    bwd += c * widths[0] + 3 * elem
    return fwd, bwd
