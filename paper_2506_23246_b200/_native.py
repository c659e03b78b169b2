"""ctypes binding of the C ABI declared in ``include/qpinn_b200.h``.

The shared library is built in-tree (``build.py``) and loaded from the
package directory.  There is no fallback: every product entry point goes
through these symbols, and a missing or unloadable library raises
``NativeLibraryError`` at first use.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors as E

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libqpinn_b200.so")

OK, ERR_CONFIG, ERR_DOMAIN, ERR_CAPACITY, ERR_INVALID_GATE, ERR_INVALID_BATCH, \
    ERR_NONFINITE, ERR_CUDA = range(8)
F32, F64 = 0, 1
LOSS_NSUMS = 23

_EXC = {
    ERR_CONFIG: E.ConfigError, ERR_DOMAIN: E.DomainError, ERR_CAPACITY: E.CapacityError,
    ERR_INVALID_GATE: E.InvalidGateError, ERR_INVALID_BATCH: E.InvalidBatchError,
    ERR_NONFINITE: E.RunAborted, ERR_CUDA: E.NativeLibraryError,
}


class LossSpec(C.Structure):
    """Mirror of ``qpinn_loss_spec``."""
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("n_local_slices", C.c_int32),
        ("slice_bin", C.c_void_p), ("slice_is_ic", C.c_void_p),
        ("eps", C.c_void_p), ("ic_target", C.c_void_p),
        ("balanced", C.c_int32), ("energy", C.c_int32), ("n_sym", C.c_int32),
        ("sym_field", C.c_int32 * 6), ("sym_axis", C.c_int32 * 6),
        ("sym_sign", C.c_double * 6),
        ("inv_count_bin", (C.c_double * 4) * 5), ("inv_count_all", C.c_double * 4),
        ("n_total", C.c_double), ("slice_size", C.c_double),
    ]


class TrunkDesc(C.Structure):
    """Mirror of ``qpinn_trunk_desc``."""
    _fields_ = [
        ("n_hidden", C.c_int32), ("rff", C.c_int32), ("hidden", C.c_int32), ("n_out", C.c_int32),
        ("off_w", C.c_int64 * 8), ("off_b", C.c_int64 * 8),
        ("off_adapter_w", C.c_int64), ("off_adapter_b", C.c_int64), ("off_tau_raw", C.c_int64),
        ("t_domain", C.c_double), ("omega", C.c_void_p),
    ]


# (name, restype, argtypes) -- exactly the symbols of include/qpinn_b200.h
_VP, _SZ, _I, _I64, _D = C.c_void_p, C.c_size_t, C.c_int, C.c_int64, C.c_double
SIGNATURES = [
    ("qpinn_last_error", C.c_char_p, []),
    ("qpinn_version", C.c_char_p, []),
    ("qpinn_circuit_create", _I, [_I, _I, _I, C.POINTER(_VP)]),
    ("qpinn_circuit_destroy", None, [_VP]),
    ("qpinn_circuit_param_count", _I, [_VP]),
    ("qpinn_circuit_n_qubits", _I, [_VP]),
    ("qpinn_circuit_dump", _SZ, [_VP, C.c_char_p, _SZ]),
    ("qpinn_circuit_plan_dump", _SZ, [_VP, C.c_char_p, _SZ]),
    ("qpinn_circuit_set_kernel_variant", _I, [_VP, _I]),
    ("qpinn_circuit_specialized", _I, [_VP]),
    ("qpinn_pqc_uses_transfer", _I, [_VP, _I]),
    ("qpinn_pqc_regime", _I, [_VP, _I, _I]),
    ("qpinn_pqc_max_qubits", _I, [_I]),
    ("qpinn_pqc_workspace_bytes", _SZ, [_VP, _I, _I64]),
    ("qpinn_pqc_state_bytes", _SZ, [_VP, _I, _I64]),
    ("qpinn_pqc_forward", _I, [_VP, _I, _I, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _SZ, _VP]),
    ("qpinn_pqc_backward", _I, [_VP, _I, _I, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                _VP, _VP, _SZ, _VP]),
    ("qpinn_pqc_forward_probe", _I, [_VP, _I, _I, _I64, _VP, _VP, _VP, _VP, _VP, _SZ, _VP]),
    ("qpinn_pqc_domain_check", _I, [_VP, _VP, C.POINTER(_D), C.POINTER(_I)]),
    ("qpinn_pqc_domain_fetch", _I, [_VP, _VP, _VP]),
    ("qpinn_pqc_domain_flags", _I, [_VP, _VP, _VP]),
    ("qpinn_loss_workspace_bytes", _SZ, [C.POINTER(LossSpec), _I, _I64]),
    ("qpinn_loss_forward_backward", _I, [C.POINTER(LossSpec), _I, _I64, _VP, _VP, _VP, _VP,
                                         _VP, _VP, _VP, _SZ, _VP]),
    ("qpinn_loss_head_forward_backward", _I, [C.POINTER(LossSpec), _I, _I64, _I, _VP, _VP, _VP,
                                              _VP, _VP, _VP, _VP, _VP, _VP, _SZ, _VP]),
    ("qpinn_loss_finalize", _I, [C.POINTER(LossSpec), _VP, _VP, _I, _D, _VP, _VP, _VP]),
    ("qpinn_trunk_workspace_bytes", _SZ, [C.POINTER(TrunkDesc), _I, _I64]),
    ("qpinn_trunk_forward", _I, [C.POINTER(TrunkDesc), _I, _I64, _VP, _VP, _VP, _VP, _VP, _VP,
                                 _SZ, _VP]),
    ("qpinn_trunk_forward_value", _I, [C.POINTER(TrunkDesc), _I, _I64, _VP, _VP, _VP, _VP, _VP,
                                       _VP, _SZ, _VP]),
    ("qpinn_trunk_backward", _I, [C.POINTER(TrunkDesc), _I, _I64, _VP, _VP, _VP, _VP, _VP, _VP,
                                  _VP, _VP, _SZ, _VP]),
    ("qpinn_adam_step", _I, [_I, _I64, _VP, _VP, _VP, _VP, _I64, _D, _D, _D, _D, _VP, _VP, _VP,
                             _VP]),
    ("qpinn_gemm_f32_workspace_bytes", _SZ, [_I, _I]),
    ("qpinn_gemm_f32", _I, [_I64, _I, _I, _VP, _I64, _VP, _I64, _VP, _I64, _VP, _SZ, _VP]),
    ("qpinn_gemm_f32_atb_workspace_bytes", _SZ, [_I64, _I, _I]),
    ("qpinn_gemm_f32_atb", _I, [_I64, _I, _I, _VP, _I64, _VP, _I64, _VP, _VP, _SZ, _VP]),
    ("qpinn_head_forward", _I, [_I, _I64, _I, _VP, _VP, _VP, _VP, _VP]),
    ("qpinn_probe_energy", _I, [_I, _I, _I64, _VP, _VP, _D, _VP, _VP]),
    ("qpinn_probe_l2", _I, [_I, _I, _I64, _VP, _VP, _VP, _VP]),
    ("qpinn_fdtd_workspace_bytes", _SZ, [_I, _I]),
    ("qpinn_fdtd_run", _I, [_I, _I, _I, _D, _I, C.POINTER(_D), _I, _D, _D, C.POINTER(C.c_int32),
                            _I, _VP, _VP, _VP, _VP, _VP, _SZ, _VP]),
]

_lib = None
_lock = threading.Lock()

# Instrumentation for bench.py: number of our kernels launched, and optional
# CUDA-event timing of named launches on the launching stream.
LAUNCHES = {"count": 0}
_TIMERS: dict = {}
_TIMING = {"on": False}


def count_launches(n: int) -> None:
    LAUNCHES["count"] += n


def timing_enabled() -> bool:
    return _TIMING["on"]


def timing(on: bool) -> None:
    _TIMING["on"] = on
    if on:
        _TIMERS.clear()


class timed:
    """Record CUDA events around a launch when timing is on."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        if _TIMING["on"]:
            import torch
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e1 = torch.cuda.Event(enable_timing=True)
            self.e0.record()
        return self

    def __exit__(self, *exc):
        if _TIMING["on"]:
            self.e1.record()
            _TIMERS.setdefault(self.name, []).append((self.e0, self.e1))
        return False


def timer_report() -> dict:
    """{name: (launches, mean ms)} for the events recorded since timing(True)."""
    out = {}
    for k, evs in _TIMERS.items():
        ms = [a.elapsed_time(b) for a, b in evs]
        out[k] = (len(ms), sum(ms) / len(ms) if ms else 0.0)
    return out


def lib():
    """Load (once) and return the native library; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise E.NativeLibraryError(
                    f"{LIB_PATH} is missing: build it with `python -m "
                    f"paper_2506_23246_b200.build` (there is no CPU fallback)")
            path = os.environ.get("QPINN_LIB_OVERRIDE", LIB_PATH)  # kernel-variant experiments
            try:
                h = C.CDLL(path)
            except OSError as e:  # pragma: no cover - depends on the box
                raise E.NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
            for name, res, args in SIGNATURES:
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    msg = lib().qpinn_last_error().decode(errors="replace")
    raise _EXC.get(rc, E.NativeLibraryError)(f"{what}: {msg}" if what else msg)


def ptr(t) -> int:
    """Device pointer of a torch tensor (or None -> NULL)."""
    return 0 if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def dtype_code(dtype) -> int:
    import torch
    if dtype == torch.float32:
        return F32
    if dtype == torch.float64:
        return F64
    raise E.ConfigError(f"unsupported dtype {dtype}; use float32 or float64")
