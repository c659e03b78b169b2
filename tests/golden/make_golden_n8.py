"""Golden LossEvaluator.evaluate(tape=True) vectors for 8-, 9-, 10- and 12-qubit hybrid
models: n = 8, 9, 10 run the transfer-matrix PQC kernels by default since round 2 (n = 8
at any depth, n = 9, 10 from L = 4; permutation, phase and two-rotation phase ansaetze);
n = 12 (strongly, L = 2) runs the multi-gate HBM passes for both K1 and K2.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_n8.py

Uses make_golden.eval_case on the reference imported from /root/reference (read-only).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402

from make_golden import ModelConfig, eval_case  # noqa: E402

w = np.array([1.0, 0.8, 0.5, 0.2, 0.05])
base = dict(variant="hybrid", hidden_width=32, rff_features=16, seed=7, t_domain=1.5)
eval_case("eval_n8_strongly.npz",
          ModelConfig(**base, n_qubits=8, n_layers_pqc=2, ansatz="strongly", scale="acos"),
          (4, 4, 5), "vacuum", chunk_slices=3, weights=w)
eval_case("eval_n9_crossmesh.npz",
          ModelConfig(**base, n_qubits=9, n_layers_pqc=4, ansatz="cross_mesh", scale="asin"),
          (4, 4, 4), "dielectric", t_end=0.7, chunk_slices=2, weights=None, energy=False)
eval_case("eval_n12_strongly.npz",
          ModelConfig(**base, n_qubits=12, n_layers_pqc=2, ansatz="strongly", scale="acos"),
          (3, 3, 3), "vacuum", chunk_slices=3, weights=w)
eval_case("eval_n10_2rot.npz",
          ModelConfig(**base, n_qubits=10, n_layers_pqc=4, ansatz="cross_mesh_2rot", scale="pi"),
          (4, 4, 3), "asymmetric", chunk_slices=2, weights=None)
