"""The reference-side ctypes binding of the B200 PQC boundary.

This is the file a ``qpinn`` maintainer would add as ``qpinn/_b200.py``. It
touches only the C ABI of ``include/qpinn_b200.h`` through ctypes; torch is
used as the device allocator and nothing from ``paper_2506_23246_b200``'s Python
package is imported. ``install(qpinn)`` swaps it in for
``qpinn.ansatz.quantum_layer_forward`` (ansatz.py:341-400) and for the name
``qpinn.network`` imported from it (network.py:25, called at :299-301), so the
reference's own ``Model.forward`` / ``LossEvaluator.evaluate(tape=True)`` run
their PQC on the B200 kernels:

* dual inputs (``BatchedDual`` of ndarrays or taped ``Tensor``\\s) ->
  ``qpinn_pqc_forward`` with x/y/t tangents; when any input is taped, one tape
  node whose VJP calls ``qpinn_pqc_backward`` (the adjoint K2) and
  accumulates into the activations, their tangents and the circuit parameters
  -- the same contract as the reference's taped ops (tape.py:84-116);
* plain inputs -> the value-only forward (a taped plain ``Tensor`` gets the
  adjoint with zero tangents);
* the reference's domain rule (ansatz.py:51-58): ``DomainError`` above
  1 + 1e-12, a clamp warning within, from the kernel's running max|a|;
* ``ConfigError`` on a wrong activation width (ansatz.py:356-357).

``tests/test_ref_binding_gpu.py`` drives the installed reference through it.
"""
from __future__ import annotations

import ctypes as C
import os
import warnings

import numpy as np
import torch

LIB_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "paper_2506_23246_b200", "libqpinn_b200.so")
_KIND = ["basic", "strongly", "cross_mesh", "cross_mesh_2rot", "cross_mesh_cnot",
         "no_entanglement"]                                   # QPINN_ANSATZ_*
_SCALE = ["none", "pi", "bias", "asin", "acos"]              # QPINN_SCALE_*
F32, F64, ERR_DOMAIN = 0, 1, 2
_vp, _sz, _i64 = C.c_void_p, C.c_size_t, C.c_int64


def _bind(lib):
    lib.qpinn_last_error.restype = C.c_char_p
    lib.qpinn_last_error.argtypes = []
    lib.qpinn_circuit_create.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]
    lib.qpinn_circuit_param_count.argtypes = [_vp]
    lib.qpinn_pqc_workspace_bytes.restype = _sz
    lib.qpinn_pqc_workspace_bytes.argtypes = [_vp, C.c_int, _i64]
    lib.qpinn_pqc_state_bytes.restype = _sz
    lib.qpinn_pqc_state_bytes.argtypes = [_vp, C.c_int, _i64]
    # 13 arguments (include/qpinn_b200.h): circuit, dtype, scale, rows, act_val,
    # act_tan, qparams, z, dz, states, workspace, workspace_bytes, stream
    lib.qpinn_pqc_forward.argtypes = [_vp, C.c_int, C.c_int, _i64] + [_vp] * 7 + [_sz, _vp]
    # 17 arguments: circuit, dtype, scale, rows, act_val, act_tan, qparams, states,
    # g_z, g_dz, g_act_val, g_act_tan, g_qparams, workspace, workspace_bytes, stream
    lib.qpinn_pqc_backward.argtypes = [_vp, C.c_int, C.c_int, _i64] + [_vp] * 10 + [_sz, _vp]
    lib.qpinn_pqc_domain_check.argtypes = [_vp, _vp, C.POINTER(C.c_double), C.POINTER(C.c_int)]
    return lib


_lib = None
_circuits = {}


def lib():
    global _lib
    if _lib is None:
        _lib = _bind(C.CDLL(LIB_PATH))
    return _lib


def _check(rc, what):
    if rc:
        raise RuntimeError(f"{what}: {lib().qpinn_last_error().decode()} (status {rc})")


def _handle(circuit):
    key = (circuit.kind.value, circuit.n_qubits, circuit.n_layers)
    h = _circuits.get(key)
    if h is None:
        h = _vp()
        _check(lib().qpinn_circuit_create(_KIND.index(key[0]), key[1], key[2], C.byref(h)),
               "qpinn_circuit_create")
        _circuits[key] = h
    return h


def _stream():
    return _vp(torch.cuda.current_stream().cuda_stream)


def _dev(x, dtype):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda")


def _p(t):
    return _vp(t.data_ptr()) if t is not None else _vp(0)


class _Call:
    """One forward on the device plus what its adjoint needs."""

    def __init__(self, circuit, scale_kind, a, da, qp, dtype, keep_states):
        L = lib()
        self.h, self.dtype = _handle(circuit), dtype
        self.code = F64 if dtype == torch.float64 else F32
        self.scale = _SCALE.index(getattr(scale_kind, "value", scale_kind))
        self.R, self.n = a.shape
        self.a, self.da, self.qp = _dev(a, dtype), (None if da is None else _dev(da, dtype)), \
            _dev(qp, dtype)
        self.ws = torch.zeros(L.qpinn_pqc_workspace_bytes(self.h, self.code, self.R),
                              dtype=torch.uint8, device="cuda")
        self.states = None
        if keep_states and da is not None:
            nb = L.qpinn_pqc_state_bytes(self.h, self.code, self.R)
            self.states = torch.empty(max(nb, 1), dtype=torch.uint8, device="cuda")
        self.z = torch.empty((self.R, self.n), dtype=dtype, device="cuda")
        self.dz = None if da is None else torch.empty((3, self.R, self.n), dtype=dtype,
                                                      device="cuda")
        _check(L.qpinn_pqc_forward(self.h, self.code, self.scale, self.R, _p(self.a),
                                   _p(self.da), _p(self.qp), _p(self.z), _p(self.dz),
                                   _p(self.states), _p(self.ws), self.ws.numel(), _stream()),
               "qpinn_pqc_forward")
        m, clamped = C.c_double(), C.c_int()
        rc = L.qpinn_pqc_domain_check(_p(self.ws), _stream(), C.byref(m), C.byref(clamped))
        if rc == ERR_DOMAIN:
            from qpinn.errors import DomainError
            raise DomainError(f"scale input exceeds [-1, 1] by {m.value - 1.0:.3e}")
        _check(rc, "qpinn_pqc_domain_check")
        if clamped.value:
            warnings.warn("scale input clamped into [-1, 1] (excursion <= 1e-12)", stacklevel=3)

    def backward(self, g_z, g_dz):
        L = lib()
        R, n = self.R, self.n
        da = self.da if self.da is not None else torch.zeros((3, R, n), dtype=self.dtype,
                                                               device="cuda")
        gz = _dev(g_z, self.dtype)
        gdz = _dev(g_dz, self.dtype) if g_dz is not None else torch.zeros_like(da)
        ga = torch.empty_like(self.a)
        gda = torch.empty_like(da)
        gq = torch.empty_like(self.qp)
        _check(L.qpinn_pqc_backward(self.h, self.code, self.scale, R, _p(self.a), _p(da),
                                    _p(self.qp), _p(self.states), _p(gz), _p(gdz), _p(ga),
                                    _p(gda), _p(gq), _p(self.ws), self.ws.numel(), _stream()),
               "qpinn_pqc_backward")
        return ga.double().cpu().numpy(), gda.double().cpu().numpy(), gq.double().cpu().numpy()


def make_quantum_layer_forward(dtype=torch.float64):
    """The drop-in for ``qpinn.ansatz.quantum_layer_forward`` (ansatz.py:341-400).

    ``via`` and ``transfer`` are accepted and ignored: the kernels choose the
    formulation (the transfer-matrix GEMM at fp32 n = 5..7, gate sweeps
    otherwise), and outputs do not depend on it."""
    from qpinn.ansatz import CircuitSpec, build_circuit
    from qpinn.autodiff.ops import BatchedDual
    from qpinn.autodiff.tape import Tensor
    from qpinn.errors import ConfigError

    def val(x):
        return x.value if isinstance(x, Tensor) else np.asarray(x, dtype=np.float64)

    def quantum_layer_forward(activations, qparams, circuit, scale_kind, via="matrix",
                              transfer=None):
        if not isinstance(circuit, CircuitSpec):
            circuit = build_circuit(circuit, n_qubits=activations.shape[1])
        n = circuit.n_qubits
        if activations.shape[1] != n:
            raise ConfigError(f"expected {n} activations per point")
        dual = isinstance(activations, BatchedDual)
        a_in = activations.val if dual else activations
        da_in = activations.tan if dual else None
        tracked = [x for x in (a_in, da_in, qparams) if isinstance(x, Tensor) and x.track]
        call = _Call(circuit, scale_kind, val(a_in), None if da_in is None else val(da_in),
                     val(qparams), dtype, keep_states=bool(tracked))
        z = call.z.double().cpu().numpy()
        if not dual:
            if not tracked:
                return z

            def vjp_plain(g):
                ga, _, gq = call.backward(np.real(g), None)
                if isinstance(a_in, Tensor):
                    a_in._accumulate(ga)
                if isinstance(qparams, Tensor):
                    qparams._accumulate(gq)
            return Tensor(z, _parents=tracked, _vjp=vjp_plain)
        dz = call.dz.double().cpu().numpy()
        if not tracked:
            return BatchedDual(z, dz)

        def vjp(g):
            g = np.real(np.asarray(g))
            ga, gda, gq = call.backward(g[0], g[1:])
            if isinstance(a_in, Tensor):
                a_in._accumulate(ga)
            if isinstance(da_in, Tensor):
                da_in._accumulate(gda)
            if isinstance(qparams, Tensor):
                qparams._accumulate(gq)
        zz = Tensor(np.concatenate([z[None], dz], axis=0), _parents=tracked, _vjp=vjp)
        return BatchedDual(zz[0], zz[1:])

    return quantum_layer_forward


def install(qpinn_module, dtype=torch.float64):
    """Patch the reference package in place; returns an ``uninstall`` callable."""
    import importlib
    ansatz = importlib.import_module(qpinn_module.__name__ + ".ansatz")
    network = importlib.import_module(qpinn_module.__name__ + ".network")
    saved = (ansatz.quantum_layer_forward, network.quantum_layer_forward)
    fn = make_quantum_layer_forward(dtype)
    ansatz.quantum_layer_forward = fn
    network.quantum_layer_forward = fn

    def uninstall():
        ansatz.quantum_layer_forward, network.quantum_layer_forward = saved
    return uninstall
