"""Golden LossEvaluator.evaluate(tape=True) vectors for 6-qubit hybrid models, which
run the transfer-matrix PQC kernels by default (one permutation and one phase ansatz).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_n6.py

Uses make_golden.eval_case on the reference imported from /root/reference (read-only).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402

from make_golden import ModelConfig, eval_case  # noqa: E402

w = np.array([1.0, 0.8, 0.5, 0.2, 0.05])
base = dict(variant="hybrid", hidden_width=32, rff_features=16, n_qubits=6, n_layers_pqc=3,
            seed=5, t_domain=1.5)
eval_case("eval_n6_strongly.npz", ModelConfig(**base, ansatz="strongly", scale="acos"),
          (4, 4, 6), "vacuum", chunk_slices=3, weights=w)
eval_case("eval_n6_crossmesh.npz", ModelConfig(**base, ansatz="cross_mesh", scale="bias"),
          (6, 4, 5), "dielectric", t_end=0.7, chunk_slices=2, weights=None, energy=False)
