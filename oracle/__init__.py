"""CPU oracle for the QPINN hot path -- TEST INFRASTRUCTURE ONLY.

This package is a plain-numpy (float64/complex128) restatement of the
reference algorithm in ``/root/reference/pkg/src/qpinn`` for the train-step
path: circuit construction and fused plan, the scaled angle embedding, the
per-point statevector circuit with forward-mode x/y/t tangents, its adjoint
backward, the dual classical trunk and its reverse pass, the fused Maxwell
loss evaluator and Adam.  Every function cites the reference file:line it
restates.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import it, and only as the checker (or as the timed CPU port).  The
product package ``paper_2506_23246_b200`` never imports it: the product path
runs the CUDA library and fails loudly when it is missing.

Parity pin: ``tests/test_oracle.py`` checks this restatement against golden
vectors produced by the reference itself (``tests/golden/make_golden.py``).
"""
from .qpinn_oracle import *  # noqa: F401,F403
