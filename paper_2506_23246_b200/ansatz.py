"""Circuit construction and the quantum layer, backed by the sm_100a kernels.

Mirrors the reference module ``qpinn.ansatz`` (ansatz.py): ``AnsatzKind``,
``ScaleKind``, ``build_circuit``, ``CircuitSpec`` (gate list, ``dump``,
``fused_plan``), ``ansatz_param_count``, ``scale`` and
``quantum_layer_forward``.  The gate schedule and fused plan are built
natively (``csrc/circuit.cu``) and parsed back here, so the kernels and the
Python view can never disagree.  ``quantum_layer_forward`` runs K1 (forward
+ x/y/t tangents) and, under autograd, K2 (adjoint backward) on CUDA tensors;
there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import warnings
import weakref
from dataclasses import dataclass, field
from enum import Enum
from typing import Optional, Tuple

import torch

from . import _native as N
from .errors import ConfigError, DomainError, InvalidGateError

CLAMP_TOL = 1e-12  # ansatz.py:24


class AnsatzKind(str, Enum):
    BASIC = "basic"
    STRONGLY = "strongly"
    CROSS_MESH = "cross_mesh"
    CROSS_MESH_2ROT = "cross_mesh_2rot"
    CROSS_MESH_CNOT = "cross_mesh_cnot"
    NO_ENTANGLEMENT = "no_entanglement"


class ScaleKind(str, Enum):
    NONE = "none"
    PI = "pi"
    BIAS = "bias"
    ASIN = "asin"
    ACOS = "acos"


_KIND_CODE = {k: i for i, k in enumerate(AnsatzKind)}
_SCALE_CODE = {k: i for i, k in enumerate(ScaleKind)}

GATE_KINDS = ("RX", "RY", "RZ", "Rot", "CNOT", "CRZ")
PARAM_COUNT = {"RX": 1, "RY": 1, "RZ": 1, "Rot": 3, "CNOT": 0, "CRZ": 1}
TWO_QUBIT = {"CNOT", "CRZ"}


@dataclass(frozen=True)
class GateOp:
    """One gate: kind, wires and slots (qsim.py:39-64)."""
    kind: str
    wires: Tuple[int, ...]
    param_slots: Tuple[int, ...] = ()
    source: str = "param"

    def __post_init__(self):
        if self.kind not in GATE_KINDS:
            raise InvalidGateError(f"unknown gate kind {self.kind!r}")
        want = 2 if self.kind in TWO_QUBIT else 1
        if len(self.wires) != want:
            raise InvalidGateError(f"{self.kind} takes {want} wire(s)")
        if len(set(self.wires)) != len(self.wires):
            raise InvalidGateError(f"wire collision in {self.kind}{self.wires}")
        if len(self.param_slots) != PARAM_COUNT[self.kind]:
            raise InvalidGateError(
                f"{self.kind} takes {PARAM_COUNT[self.kind]} parameter slot(s)")
        if self.source not in ("param", "embed"):
            raise InvalidGateError(f"bad slot source {self.source!r}")


def _read_text(fn, handle) -> str:
    n = fn(handle, None, 0)
    buf = C.create_string_buffer(n)
    fn(handle, buf, n)
    return buf.value.decode()


class CircuitSpec:
    """Ordered gate list (embedding first) and its fused execution plan.

    Immutable after construction (ansatz.py:70-109).  Owns the native plan
    handle; the device copy is uploaded lazily on first kernel launch.
    """

    def __init__(self, kind: AnsatzKind, n_qubits: int, n_layers: int):
        lib = N.lib()
        h = C.c_void_p()
        N.check(lib.qpinn_circuit_create(_KIND_CODE[kind], n_qubits, n_layers, C.byref(h)),
                "build_circuit")
        self._h = h
        self.kind = kind
        self.n_qubits = n_qubits
        self.n_layers = n_layers
        self.param_count = lib.qpinn_circuit_param_count(h)
        self._dump = _read_text(lib.qpinn_circuit_dump, h)
        self._plan_text = _read_text(lib.qpinn_circuit_plan_dump, h)
        self.gates = tuple(self._parse_gate(line) for line in self._dump.splitlines())
        self._workspaces: dict = {}

    @staticmethod
    def _parse_gate(line: str) -> GateOp:
        kind, wires, slots = line.split(" ")
        w = tuple(int(v) for v in wires.split(","))
        if slots == "-":
            return GateOp(kind, w)
        src, idx = slots.split(":")
        return GateOp(kind, w, tuple(int(v) for v in idx.split(",")),
                      "embed" if src == "embed" else "param")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and N._lib is not None:
            N._lib.qpinn_circuit_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def embed_gates(self):
        return self.gates[:self.n_qubits]

    @property
    def layer_gates(self):
        return self.gates[self.n_qubits:]

    def dump(self) -> str:
        """Plain-text gate list, one gate per line (ansatz.py:98-109)."""
        return self._dump

    def fused_plan(self) -> list:
        """Fused steps as parsed from the native plan (ansatz.py:93-96, :117-156):
        ("u1", kind, wire, slots) | ("perm", [perm...]) | ("phases", [(c, t, slot)...])."""
        out = []
        for line in self._plan_text.splitlines():
            tag, rest = line.split(" ", 1)
            if tag == "u1":
                kind, wire, slots = rest.split(" ")
                out.append(("u1", kind, int(wire), tuple(int(s) for s in slots.split(","))))
            elif tag == "perm":
                out.append(("perm", [int(v) for v in rest.split(",")]))
            else:
                out.append(("phases", [tuple(int(v) for v in p.split(":"))
                                       for p in rest.split(" ")]))
        return out

    def workspace(self, dtype, device, rows: int) -> torch.Tensor:
        """Cached device scratch for K1/K2 (grown on demand)."""
        need = N.lib().qpinn_pqc_workspace_bytes(self._h, N.dtype_code(dtype), rows)
        device = torch.device(device)
        if device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        key = (dtype, str(device))
        ws = self._workspaces.get(key)
        if ws is None or ws.numel() < need:
            grown = torch.zeros(need, dtype=torch.uint8, device=device)
            if ws is not None:  # keep the running max|a| of forwards not yet checked
                grown[:8].copy_(ws[:8])
            ws = grown
            self._workspaces[key] = ws
        return ws

    @property
    def specialized(self) -> bool:
        """Compile-time specialised K1/K2 exist for this (ansatz, n, L)."""
        return bool(N.lib().qpinn_circuit_specialized(self._h))

    def uses_transfer(self, dtype) -> bool:
        """K1/K2 run as the transfer-matrix map on the tensor cores for ``dtype``."""
        return bool(N.lib().qpinn_pqc_uses_transfer(self._h, N.dtype_code(dtype)))

    REGIMES = ("layer", "generic", "transfer", "cta/cluster", "multi-gate HBM", "global")

    def regime(self, dtype, backward: bool = False) -> str:
        """The kernels K1 (or, with backward, K2) runs for this circuit and dtype."""
        r = N.lib().qpinn_pqc_regime(self._h, N.dtype_code(dtype), int(backward))
        return self.REGIMES[r] if 0 <= r < len(self.REGIMES) else "unknown"

    def set_kernel_variant(self, variant: str) -> None:
        """"auto" (transfer-matrix kernels for float32 n = 5..8, and n = 9, 10 from
        L = 4, else the layer-loop / CTA kernels), "generic", "transfer" (float32,
        5 <= n <= 10: the transfer-matrix map on the tensor cores) or "layer"
        (the layer-loop kernels wherever they apply)."""
        code = {"auto": 0, "generic": 1, "transfer": 2, "layer": 3}[variant]
        N.check(N.lib().qpinn_circuit_set_kernel_variant(self._h, code), "set_kernel_variant")

    def __repr__(self):
        return (f"CircuitSpec(kind={self.kind.value}, n_qubits={self.n_qubits}, "
                f"n_layers={self.n_layers}, param_count={self.param_count})")


def build_circuit(kind: AnsatzKind | str, n_qubits: int = 7, n_layers: int = 4) -> CircuitSpec:
    """ansatz.py:159-207 (native builder)."""
    try:
        kind = AnsatzKind(kind)
    except ValueError as e:
        raise ConfigError(str(e)) from e
    return CircuitSpec(kind, n_qubits, n_layers)


def ansatz_param_count(kind: AnsatzKind | str, n_qubits: int = 7, n_layers: int = 4) -> int:
    return build_circuit(kind, n_qubits, n_layers).param_count


class BatchedDual:
    """Value [R, ...] plus three input tangents [3, R, ...] (ops.py:64-132)."""

    __slots__ = ("val", "tan")

    def __init__(self, val, tan):
        self.val = val
        self.tan = tan

    @property
    def shape(self):
        return self.val.shape

    def __repr__(self):
        return f"BatchedDual(shape={tuple(self.val.shape)})"


def scale(kind: ScaleKind | str, a: torch.Tensor) -> torch.Tensor:
    """Activation in [-1, 1] -> embedding angle (ansatz.py:44-67).

    Utility mirror of the reference function (the kernels fuse it); same
    DomainError / clamp-with-warning semantics.
    """
    kind = ScaleKind(kind)
    if a.numel():
        over = float(a.abs().max()) - 1.0
        if over > CLAMP_TOL:
            raise DomainError(f"scale input exceeds [-1, 1] by {over:.3e}")
        if over > 0.0:
            warnings.warn("scale input clamped into [-1, 1] (excursion <= 1e-12)", stacklevel=2)
            a = a.clamp(-1.0, 1.0)
    if kind is ScaleKind.NONE:
        return a
    if kind is ScaleKind.PI:
        return a * torch.pi
    if kind is ScaleKind.BIAS:
        return (a + 1.0) * (torch.pi / 2.0)
    if kind is ScaleKind.ASIN:
        return torch.asin(a) + torch.pi / 2.0
    return torch.acos(a)


def _check_rows(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ConfigError(f"{name} must be a CUDA tensor (the kernels have no CPU path)")


def check_domain(circuit: CircuitSpec, dtype, device, stream=None, ws=None) -> float:
    """Synchronise and apply the reference domain rule (ansatz.py:51-58) to the
    forwards launched on ``circuit``'s workspace (or ``ws``) since the last
    check; returns max|a|."""
    ws = circuit.workspace(dtype, device, 0) if ws is None else ws
    m = C.c_double()
    clamped = C.c_int()
    rc = N.lib().qpinn_pqc_domain_check(C.c_void_p(ws.data_ptr()),
                                        C.c_void_p(N.stream_ptr(stream)),
                                        C.byref(m), C.byref(clamped))
    if rc == N.ERR_DOMAIN:
        raise DomainError(f"scale input exceeds [-1, 1] by {m.value - 1.0:.3e}")
    N.check(rc, "domain check")
    if clamped.value:
        warnings.warn("scale input clamped into [-1, 1] (excursion <= 1e-12)", stacklevel=3)
    return m.value


def domain_rule(m: float) -> None:
    """The reference domain rule (ansatz.py:51-58) on a fetched max|a|."""
    over = m - 1.0
    if over > 1e-12:
        raise DomainError(f"scale input exceeds [-1, 1] by {over:.3e}")
    if over > 0.0:
        warnings.warn("scale input clamped into [-1, 1] (excursion <= 1e-12)", stacklevel=3)


def state_buffer(circuit: CircuitSpec, a) -> torch.Tensor:
    """Final-state hand-off buffer K1 -> K2 (4 states x 2^n complex per row)."""
    nbytes = N.lib().qpinn_pqc_state_bytes(circuit.handle, N.dtype_code(a.dtype), a.shape[0])
    return torch.empty(nbytes // a.element_size(), dtype=a.dtype, device=a.device)


def pqc_forward_raw(circuit: CircuitSpec, scale_kind, a, da, qp, states=None):
    """K1 launch: z [R,n] and dz [3,R,n] (dz None when da is None); fills
    ``states`` (see ``state_buffer``) for the backward when given."""
    R, n = a.shape
    z = torch.empty_like(a)
    dz = torch.empty((3, R, n), dtype=a.dtype, device=a.device) if da is not None else None
    ws = circuit.workspace(a.dtype, a.device, R)
    with N.timed("pqc_forward"):
        rc = N.lib().qpinn_pqc_forward(
            circuit.handle, N.dtype_code(a.dtype), _SCALE_CODE[ScaleKind(scale_kind)], R,
            N.ptr(a), N.ptr(da), N.ptr(qp), N.ptr(z), N.ptr(dz), N.ptr(states), ws.data_ptr(),
            ws.numel(), N.stream_ptr())
    N.check(rc, "qpinn_pqc_forward")
    N.count_launches(1 if R else 0)
    return z, dz


def pqc_backward_raw(circuit: CircuitSpec, scale_kind, a, da, qp, gz, gdz, states=None):
    """K2 launch: (g_a [R,n], g_da [3,R,n], g_qp [P]); ``states`` from the
    matching forward skips the circuit replay."""
    R, n = a.shape
    ga = torch.empty_like(a)
    gda = torch.empty_like(da)
    gq = torch.empty_like(qp)
    ws = circuit.workspace(a.dtype, a.device, R)
    with N.timed("pqc_backward"):
        rc = N.lib().qpinn_pqc_backward(
            circuit.handle, N.dtype_code(a.dtype), _SCALE_CODE[ScaleKind(scale_kind)], R,
            N.ptr(a), N.ptr(da), N.ptr(qp), N.ptr(states), N.ptr(gz), N.ptr(gdz), N.ptr(ga),
            N.ptr(gda), N.ptr(gq), ws.data_ptr(), ws.numel(), N.stream_ptr())
    N.check(rc, "qpinn_pqc_backward")
    N.count_launches(3 if R else 0)
    return ga, gda, gq


# -- torch custom ops (SURVEY §8 b): torch.ops.qpinn_b200.pqc_fwd_tangent / pqc_bwd_adjoint --
#
# The plan descriptor crosses the op boundary as an integer token for a live
# CircuitSpec (ops schemas carry tensors and scalars only); the K1 -> K2 state
# hand-off is an ordinary tensor output, so the ops are functional.

_PLANS: "weakref.WeakValueDictionary[int, CircuitSpec]" = weakref.WeakValueDictionary()


def plan_token(circuit: CircuitSpec) -> int:
    """Integer handle of ``circuit`` for the ``torch.ops.qpinn_b200`` schemas."""
    tok = id(circuit)
    _PLANS[tok] = circuit
    return tok


def _plan(tok: int) -> CircuitSpec:
    c = _PLANS.get(tok)
    if c is None:
        raise ConfigError(f"unknown circuit plan token {tok}")
    return c


@torch.library.custom_op("qpinn_b200::pqc_fwd_tangent", mutates_args=())
def pqc_fwd_tangent(plan: int, scale_kind: str, act_val: torch.Tensor, act_tan: torch.Tensor,
                    qparams: torch.Tensor, save_states: bool
                    ) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """K1: (z [R,n], dz [3,R,n], states); ``states`` is empty unless
    ``save_states`` (ansatz.py:341-400)."""
    c = _plan(plan)
    states = (state_buffer(c, act_val) if save_states
              else act_val.new_empty(0))
    z, dz = pqc_forward_raw(c, scale_kind, act_val, act_tan, qparams,
                            states if save_states else None)
    return z, dz, states


@pqc_fwd_tangent.register_fake
def _(plan, scale_kind, act_val, act_tan, qparams, save_states):
    c = _plan(plan)
    n_states = 0
    if save_states:
        nbytes = N.lib().qpinn_pqc_state_bytes(c.handle, N.dtype_code(act_val.dtype),
                                              act_val.shape[0])
        n_states = nbytes // act_val.element_size()
    return (torch.empty_like(act_val), torch.empty_like(act_tan),
            act_val.new_empty(n_states))


@torch.library.custom_op("qpinn_b200::pqc_bwd_adjoint", mutates_args=())
def pqc_bwd_adjoint(plan: int, scale_kind: str, act_val: torch.Tensor, act_tan: torch.Tensor,
                    qparams: torch.Tensor, states: torch.Tensor, g_z: torch.Tensor,
                    g_dz: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """K2: (g_act_val [R,n], g_act_tan [3,R,n], g_qparams [P]); an empty
    ``states`` replays the circuit instead of reading the K1 hand-off."""
    return pqc_backward_raw(_plan(plan), scale_kind, act_val, act_tan, qparams,
                            g_z.contiguous(), g_dz.contiguous(),
                            states if states.numel() else None)


@pqc_bwd_adjoint.register_fake
def _(plan, scale_kind, act_val, act_tan, qparams, states, g_z, g_dz):
    return torch.empty_like(act_val), torch.empty_like(act_tan), torch.empty_like(qparams)


def _fwd_setup_context(ctx, inputs, output):
    plan, scale_kind, a, da, qp, _ = inputs
    ctx.plan, ctx.scale_kind = plan, scale_kind
    ctx.save_for_backward(a, da, qp, output[2])


def _fwd_backward(ctx, gz, gdz, _gstates):
    a, da, qp, states = ctx.saved_tensors
    gz = torch.zeros_like(a) if gz is None else gz
    gdz = torch.zeros_like(da) if gdz is None else gdz
    ga, gda, gq = torch.ops.qpinn_b200.pqc_bwd_adjoint(ctx.plan, ctx.scale_kind, a, da, qp,
                                                       states, gz, gdz)
    return None, None, ga, gda, gq, None


pqc_fwd_tangent.register_autograd(_fwd_backward, setup_context=_fwd_setup_context)


class _PQCValue(torch.autograd.Function):
    """Value-only K1 (no tangents).  Its backward reuses K2 with zero tangents."""

    @staticmethod
    def forward(ctx, a, qp, circuit, scale_kind):
        z, _ = pqc_forward_raw(circuit, scale_kind, a, None, qp)
        ctx.save_for_backward(a, qp)
        ctx.circuit = circuit
        ctx.scale_kind = scale_kind
        return z

    @staticmethod
    def backward(ctx, gz):
        a, qp = ctx.saved_tensors
        da = torch.zeros((3,) + tuple(a.shape), dtype=a.dtype, device=a.device)
        ga, _, gq = pqc_backward_raw(ctx.circuit, ctx.scale_kind, a, da, qp, gz.contiguous(),
                                     torch.zeros_like(da))
        return ga, gq, None, None


def quantum_layer_forward(activations, qparams, circuit: CircuitSpec | AnsatzKind | str,
                          scale_kind: ScaleKind | str, via: str = "kernel", transfer=None,
                          check: bool = True):
    """Scaled angle embedding -> PQC -> per-qubit <Z> (ansatz.py:341-400).

    ``activations`` is a CUDA tensor [R, n] or a ``BatchedDual`` (val [R,n],
    tan [3,R,n]); returns the same kind.  Differentiable through autograd
    (values, tangents and ``qparams``).  ``via``/``transfer`` are accepted for
    signature compatibility; the kernel path applies the gates directly.
    ``check`` synchronises to apply the reference's DomainError rule; the
    training engine passes False and checks once per step instead.
    """
    del transfer
    if via not in ("kernel", "matrix", "gates"):
        raise ConfigError(f"unknown via {via!r}")
    dual = isinstance(activations, BatchedDual)
    a = activations.val if dual else activations
    if not isinstance(circuit, CircuitSpec):
        circuit = build_circuit(circuit, n_qubits=a.shape[1])
    n = circuit.n_qubits
    if a.dim() != 2 or a.shape[1] != n:
        raise ConfigError(f"expected {n} activations per point")
    _check_rows(a, "activations")
    qp = qparams
    if not torch.is_tensor(qp):
        qp = torch.as_tensor(qp, dtype=a.dtype, device=a.device)
    if qp.numel() != circuit.param_count:
        raise ConfigError(f"expected {circuit.param_count} circuit parameters")
    a = a.contiguous()
    qp = qp.to(dtype=a.dtype).contiguous()
    if dual:
        da = activations.tan.to(dtype=a.dtype).contiguous()
        if tuple(da.shape) != (3,) + tuple(a.shape):
            raise ConfigError("activation tangents must have shape [3, R, n]")
        save = torch.is_grad_enabled() and (a.requires_grad or da.requires_grad
                                            or qp.requires_grad)
        z, dz, _ = torch.ops.qpinn_b200.pqc_fwd_tangent(
            plan_token(circuit), ScaleKind(scale_kind).value, a, da, qp, save)
        if check:
            check_domain(circuit, a.dtype, a.device)
        return BatchedDual(z, dz)
    z = _PQCValue.apply(a, qp, circuit, ScaleKind(scale_kind))
    if check:
        check_domain(circuit, a.dtype, a.device)
    return z
