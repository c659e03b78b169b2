"""B200-native QPINN hot path (arXiv 2506.23246).

Drop-in for the reference ``qpinn`` train-step path: circuit construction,
the per-point PQC with forward-mode x/y/t tangents and its adjoint backward
(hand-written sm_100a kernels behind the C ABI in ``include/qpinn_b200.h``),
the fused Maxwell loss, Adam and the device-resident epoch engine.
"""
import torch as _torch

# the reference computes in float64; the float32 build must not silently
# drop to TF32 inside the trunk GEMMs
_torch.backends.cuda.matmul.allow_tf32 = False
_torch.backends.cudnn.allow_tf32 = False

from .errors import (CapacityError, ConfigError, ContractViolation, DomainError,  # noqa: E402
                     InvalidBatchError, InvalidGateError, MetricError, NativeLibraryError,
                     QpinnError, RunAborted)
from .ansatz import (AnsatzKind, BatchedDual, CircuitSpec, GateOp, ScaleKind,  # noqa: E402
                     ansatz_param_count, build_circuit, quantum_layer_forward, scale)

__all__ = [
    "AnsatzKind", "ScaleKind", "GateOp", "CircuitSpec", "BatchedDual", "build_circuit",
    "ansatz_param_count", "quantum_layer_forward", "scale", "QpinnError", "ConfigError",
    "DomainError", "CapacityError", "InvalidGateError", "InvalidBatchError", "MetricError",
    "ContractViolation", "RunAborted", "NativeLibraryError",
]
