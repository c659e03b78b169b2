"""numpy float64 restatement of the reference QPINN train-step path (test oracle).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Nothing in the
product package imports this module.

All citations are ``/root/reference/pkg/src/qpinn/<file>:<line>``.  The
restatement is deliberately independent of the reference's implementation
strategy: the circuit runs gate by gate on a [states, R, 2^n] array (the
reference uses a transfer matrix), and gradients come from hand-derived
reverse passes (the reference uses its numpy tape), so agreement with the
reference's golden vectors is a genuine cross-check.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "KINDS", "SCALES", "OracleError", "build_circuit", "fused_plan",
    "permutation_for_cnots", "crz_mesh_phase_matrix", "u1_matrix", "u1_dmatrices",
    "scale_derivs", "pqc_forward", "pqc_backward", "OracleModel", "Grid",
    "Evaluator", "time_bin_weights", "lr_at", "adam_update", "init_quantum_params",
    "train_curve", "pqc_state", "meyer_wallach", "model_predict", "adapter_activations",
    "probe_entanglement", "epsilon_at", "total_energy", "energy_probe", "bh_index",
    "l2_against_reference", "fdtd_run",
]

KINDS = ("basic", "strongly", "cross_mesh", "cross_mesh_2rot", "cross_mesh_cnot",
         "no_entanglement")
SCALES = ("none", "pi", "bias", "asin", "acos")
CLAMP_TOL = 1e-12  # ansatz.py:24


class OracleError(Exception):
    pass


# -- circuit construction (ansatz.py:112-207, qsim.py:182-225) --------------------

def build_circuit(kind: str, n: int, L: int):
    """Gate list [(kind, wires, slots, source)] and param count; ansatz.py:159-207."""
    if kind not in KINDS:
        raise OracleError(kind)
    gates = [("RX", (q,), (q,), "embed") for q in range(n)]
    slot = 0

    def take(k):
        nonlocal slot
        out = tuple(range(slot, slot + k))
        slot += k
        return out

    mesh = [(i, j) for i in range(n) for j in range(n) if j != i]  # ansatz.py:112-114
    for layer in range(1, L + 1):
        if kind in ("basic", "strongly", "cross_mesh_cnot", "no_entanglement"):
            for q in range(n):
                gates.append(("Rot", (q,), take(3), "param"))
        elif kind == "cross_mesh":
            for q in range(n):
                gates.append(("RX", (q,), take(1), "param"))
        else:
            for q in range(n):
                gates.append(("RX", (q,), take(1), "param"))
                gates.append(("RZ", (q,), take(1), "param"))
        if kind == "basic":
            gates += [("CNOT", (i, (i + 1) % n), (), "param") for i in range(n)]
        elif kind == "strongly":
            gap = (layer - 1) % (n - 1) + 1  # ansatz.py:196
            gates += [("CNOT", (i, (i + gap) % n), (), "param") for i in range(n)]
        elif kind == "cross_mesh_cnot":
            gates += [("CNOT", p, (), "param") for p in mesh]
        elif kind in ("cross_mesh", "cross_mesh_2rot"):
            gates += [("CRZ", p, take(1), "param") for p in mesh]
    return gates, slot


def permutation_for_cnots(pairs, n):
    """new[:, j] = old[:, perm[j]]; qsim.py:182-195."""
    idx = np.arange(2 ** n)
    perm = idx.copy()
    for c, t in pairs:
        on = ((idx >> (n - 1 - c)) & 1).astype(bool)
        sigma = np.where(on, idx ^ (1 << (n - 1 - t)), idx)
        perm = perm[sigma]
    return perm


def crz_mesh_phase_matrix(pairs, n):
    """[2^n, len(pairs)] phase exponents; qsim.py:212-225."""
    idx = np.arange(2 ** n)
    cols = []
    for c, t in pairs:
        on = ((idx >> (n - 1 - c)) & 1).astype(np.float64)
        tb = ((idx >> (n - 1 - t)) & 1).astype(np.float64)
        cols.append(on * (tb - 0.5))
    return np.stack(cols, axis=1)


def fused_plan(gates, n):
    """Fuse layer gates into (u1|perm|phases) steps; ansatz.py:117-156."""
    layer = [g for g in gates if g[3] != "embed"]
    steps = []
    i = 0
    while i < len(layer):
        k, w, s, src = layer[i]
        if k == "CNOT":
            j = i
            while j < len(layer) and layer[j][0] == "CNOT":
                j += 1
            steps.append(("perm", permutation_for_cnots([g[1] for g in layer[i:j]], n)))
            i = j
        elif k == "CRZ":
            j = i
            while j < len(layer) and layer[j][0] == "CRZ":
                j += 1
            run = layer[i:j]
            steps.append(("phases", crz_mesh_phase_matrix([g[1] for g in run], n),
                          np.array([g[2][0] for g in run])))
            i = j
        elif (k == "RX" and i + 1 < len(layer) and layer[i + 1][0] == "RZ"
              and layer[i + 1][1] == w):
            steps.append(("u1", "rxrz", w[0], (s[0], layer[i + 1][2][0])))
            i += 2
        else:
            steps.append(("u1", k.lower(), w[0], s))
            i += 1
    return steps


# -- gate matrices (qsim.py:274-316) and their parameter derivatives --------------

def _rx(t):
    c, s = math.cos(t / 2), math.sin(t / 2)
    return np.array([[c, -1j * s], [-1j * s, c]])


def _drx(t):
    c, s = math.cos(t / 2), math.sin(t / 2)
    return 0.5 * np.array([[-s, -1j * c], [-1j * c, -s]])


def _ry(t):
    c, s = math.cos(t / 2), math.sin(t / 2)
    return np.array([[c, -s], [s, c]], dtype=complex)


def _dry(t):
    c, s = math.cos(t / 2), math.sin(t / 2)
    return 0.5 * np.array([[-s, -c], [c, -s]], dtype=complex)


def _rz(t):
    return np.array([[np.exp(-0.5j * t), 0], [0, np.exp(0.5j * t)]])


def _drz(t):
    return np.array([[-0.5j * np.exp(-0.5j * t), 0], [0, 0.5j * np.exp(0.5j * t)]])


def u1_matrix(kind, th):
    """2x2 matrix of a fused single-qubit step; Rot = RZ(c)RY(b)RZ(a) (qsim.py:294-305),
    rxrz = RZ(b)RX(a) (qsim.py:308-316)."""
    if kind == "rot":
        return _rz(th[2]) @ _ry(th[1]) @ _rz(th[0])
    if kind == "rxrz":
        return _rz(th[1]) @ _rx(th[0])
    return {"rx": _rx, "ry": _ry, "rz": _rz}[kind](th[0])


def u1_dmatrices(kind, th):
    """d(matrix)/d(slot) for every slot of the step, in slot order."""
    if kind == "rot":
        a, b, c = th
        return [_rz(c) @ _ry(b) @ _drz(a), _rz(c) @ _dry(b) @ _rz(a),
                _drz(c) @ _ry(b) @ _rz(a)]
    if kind == "rxrz":
        return [_rz(th[1]) @ _drx(th[0]), _drz(th[1]) @ _rx(th[0])]
    return [{"rx": _drx, "ry": _dry, "rz": _drz}[kind](th[0])]


# -- scaling (ansatz.py:44-67, ops.py:181-192, ops.py:217-223) --------------------

def scale_derivs(kind, a):
    """theta = S(a), S'(a), S''(a); DomainError semantics of ansatz.py:51-58."""
    a = np.asarray(a, dtype=np.float64)
    over = np.max(np.abs(a)) - 1.0 if a.size else 0.0
    if over > CLAMP_TOL:
        raise OracleError(f"scale input exceeds [-1, 1] by {over:.3e}")
    if over > 0.0:
        a = np.clip(a, -1.0, 1.0)
    z = np.zeros_like(a)
    if kind == "none":
        return a.copy(), z + 1.0, z
    if kind == "pi":
        return a * np.pi, z + np.pi, z
    if kind == "bias":
        return (a + 1.0) * (np.pi / 2.0), z + np.pi / 2.0, z
    r = np.sqrt(1.0 - a * a)
    if kind == "asin":
        return np.arcsin(a) + np.pi / 2.0, 1.0 / r, a / (r * r * r)
    if kind == "acos":
        return np.arccos(a), -1.0 / r, -a / (r * r * r)
    raise OracleError(kind)


# -- statevector circuit with tangents -------------------------------------------

def _apply_u(states, n, q, U):
    """2x2 on wire q (wire 0 = MSB, qsim.py:5-6) of [..., 2^n] arrays."""
    sh = states.shape
    s4 = states.reshape(sh[:-1] + (2 ** q, 2, 2 ** (n - q - 1)))
    out = np.einsum("ij,...ljt->...lit", U, s4)
    return out.reshape(sh)


def _flip(states, n, q):
    idx = np.arange(2 ** n) ^ (1 << (n - 1 - q))
    return states[..., idx]


def _signs(n):
    idx = np.arange(2 ** n)
    return np.stack([1.0 - 2.0 * ((idx >> (n - 1 - q)) & 1) for q in range(n)], axis=1)


def _product_state(theta, n):
    """prod_q RX(theta_q)|0>, wire 0 the MSB; ansatz.py:233-243."""
    R = theta.shape[0]
    amp = np.ones((R, 1), dtype=np.complex128)
    for q in range(n):
        c = np.cos(0.5 * theta[:, q])[:, None]
        s = np.sin(0.5 * theta[:, q])[:, None]
        amp = np.stack([amp * c, amp * (-1j * s)], axis=2).reshape(R, -1)
    return amp


def _step_params(step, qp):
    return np.array([qp[s] for s in step[3]])


def _run_steps(states, n, steps, qp):
    for st in steps:
        if st[0] == "perm":
            states = states[..., st[1]]
        elif st[0] == "phases":
            phi = st[1] @ qp[st[2]]
            states = states * np.exp(1j * phi)
        else:
            states = _apply_u(states, n, st[2], u1_matrix(st[1], _step_params(st, qp)))
    return states


def pqc_forward(a, da, qp, kind, scale, n_layers):
    """quantum_layer_forward on a dual input; ansatz.py:341-400.

    a [R,n], da [3,R,n] (or None) -> z [R,n], dz [3,R,n] (or None).
    """
    a = np.asarray(a, dtype=np.float64)
    R, n = a.shape
    gates, P = build_circuit(kind, n, n_layers)
    if len(qp) != P:
        raise OracleError("qparams length")
    steps = fused_plan(gates, n)
    theta, s1, _ = scale_derivs(scale, a)
    phi = _product_state(theta, n)
    sign = _signs(n)
    if da is None:
        psi = _run_steps(phi, n, steps, qp)
        return (psi.real ** 2 + psi.imag ** 2) @ sign, None
    dth = s1[None] * np.asarray(da, dtype=np.float64)  # [3,R,n]
    tans = np.zeros((3, R, 2 ** n), dtype=np.complex128)
    for q in range(n):
        xq = _flip(phi, n, q)
        tans += (-0.5j) * dth[:, :, q, None] * xq[None]
    st = np.concatenate([phi[None], tans], axis=0)
    st = _run_steps(st, n, steps, qp)
    psi = st[0]
    z = (psi.real ** 2 + psi.imag ** 2) @ sign
    dz = np.stack([(2.0 * np.real(np.conj(psi) * st[k + 1])) @ sign for k in range(3)])
    return z, dz


def pqc_backward(a, da, qp, kind, scale, n_layers, gz, gdz):
    """Adjoint-differentiation backward of ``pqc_forward``.

    Returns (g_a [R,n], g_da [3,R,n], g_qp [P]).  Complex adjoints follow the
    reference's Wirtinger convention dL/dRe + i dL/dIm (tape.py:5-9).
    """
    a = np.asarray(a, dtype=np.float64)
    da = np.asarray(da, dtype=np.float64)
    R, n = a.shape
    gates, P = build_circuit(kind, n, n_layers)
    steps = fused_plan(gates, n)
    theta, s1, s2 = scale_derivs(scale, a)
    phi = _product_state(theta, n)
    dth = s1[None] * da
    tans = np.zeros((3, R, 2 ** n), dtype=np.complex128)
    for q in range(n):
        tans += (-0.5j) * dth[:, :, q, None] * _flip(phi, n, q)[None]
    x = _run_steps(np.concatenate([phi[None], tans], axis=0), n, steps, qp)
    sign = _signs(n)
    w = np.asarray(gz) @ sign.T                      # [R,D]
    v = np.einsum("krq,bq->krb", np.asarray(gdz), sign)  # [3,R,D]
    adj = np.empty_like(x)
    adj[0] = 2.0 * w * x[0] + 2.0 * np.sum(v * x[1:], axis=0)
    adj[1:] = 2.0 * v * x[0][None]
    gq = np.zeros(P)
    for st in reversed(steps):
        if st[0] == "perm":
            inv = np.empty_like(st[1])
            inv[st[1]] = np.arange(len(st[1]))
            x = x[..., inv]
            adj = adj[..., inv]
        elif st[0] == "phases":
            pmat, slots = st[1], st[2]
            ph = np.exp(1j * (pmat @ qp[slots]))
            pb = np.sum(np.conj(adj) * 1j * x, axis=0).real.sum(axis=0)  # [D]
            gq[slots] += pb @ pmat
            x = x * np.conj(ph)
            adj = adj * np.conj(ph)
        else:
            kindu, q, slots = st[1], st[2], st[3]
            th = _step_params(st, qp)
            U = u1_matrix(kindu, th)
            Uh = U.conj().T
            x = _apply_u(x, n, q, Uh)
            sh = x.shape
            x4 = x.reshape(sh[:-1] + (2 ** q, 2, 2 ** (n - q - 1)))
            a4 = adj.reshape(x4.shape)
            M = np.einsum("srlit,srljt->ij", np.conj(a4), x4)
            for s, dU in zip(slots, u1_dmatrices(kindu, th)):
                gq[s] += np.real(np.sum(dU * M))
            adj = _apply_u(adj, n, q, Uh)
    phib, mu = adj[0], adj[1:]
    rho = np.zeros_like(mu)
    for q in range(n):
        rho += dth[:, :, q, None] * _flip(mu, n, q)
    eta = 0.5j * phib - 0.25 * np.sum(rho, axis=0)
    g_th = np.zeros((R, n))
    g_dth = np.zeros((3, R, n))
    for q in range(n):
        xq = _flip(phi, n, q)
        g_th[:, q] = np.real(np.sum(np.conj(eta) * xq, axis=-1))
        g_dth[:, :, q] = np.real(np.sum(np.conj(0.5j * mu) * xq[None], axis=-1))
    g_a = g_th * s1 + np.sum(g_dth * da, axis=0) * s2
    g_da = g_dth * s1[None]
    return g_a, g_da, gq


# -- model (network.py) --------------------------------------------------------

VARIANTS = ("classical_regular", "classical_reduced", "classical_extra", "hybrid")
N_HIDDEN = {"classical_regular": 4, "classical_reduced": 3, "classical_extra": 5}
TAU_RAW_INIT = float(np.log(np.e - 1.0))  # network.py:33


@dataclass
class OracleModel:
    """Flat layout + init + dual forward/backward of network.py:180-339."""
    variant: str = "hybrid"
    hidden: int = 128
    rff: int = 128
    n_qubits: int = 7
    n_layers: int = 4
    ansatz: Optional[str] = "strongly"
    scale: Optional[str] = "acos"
    sigma: float = 1.0
    seed: int = 0
    t_domain: float = 1.5

    def __post_init__(self):
        h, win = self.hidden, 2 * self.rff
        dims = [(win, h)]
        if self.variant == "hybrid":
            dims += [(h, h), (h, h)]
            _, self.n_quantum = build_circuit(self.ansatz, self.n_qubits, self.n_layers)
            adapter, out = (h, self.n_qubits), (self.n_qubits, 3)
        else:
            dims += [(h, h)] * (N_HIDDEN[self.variant] - 1)
            self.n_quantum, adapter, out = 0, None, (h, 3)
        layout, off = [], 0
        for name, shape in ([(f"h{i}.{p}", s) for i, (fi, fo) in enumerate(dims)
                             for p, s in (("W", (fi, fo)), ("b", (fo,)))]
                            + ([("adapter.W", adapter), ("adapter.b", (adapter[1],))]
                               if adapter else [])
                            + [("out.W", out), ("out.b", (3,)), ("tau_raw", ())]):
            layout.append((name, off, shape))
            off += int(np.prod(shape, dtype=int))
        self.n_classical = off
        if self.n_quantum:
            layout.append(("quantum", off, (self.n_quantum,)))
            off += self.n_quantum
        self.layout = layout
        self.n_total = off
        self.n_hidden = len(dims)
        self.omega = np.random.default_rng([self.seed, 0]).normal(
            0.0, self.sigma, size=(self.rff, 6))  # network.py:228-230

    def init_params(self):
        """network.py:238-255."""
        rng = np.random.default_rng([self.seed, 1])
        flat = np.zeros(self.n_total)
        for name, off, shape in self.layout:
            size = int(np.prod(shape, dtype=int))
            if name.endswith(".W"):
                lim = np.sqrt(6.0 / (shape[0] + shape[1]))
                flat[off:off + size] = rng.uniform(-lim, lim, size)
            elif name == "tau_raw":
                flat[off] = TAU_RAW_INIT
        if self.n_quantum:
            flat[self.n_classical:] = np.random.default_rng([self.seed, 2]).uniform(
                0.0, 2.0 * np.pi, self.n_quantum)
        return flat

    def views(self, flat):
        return {name: flat[off:off + int(np.prod(shape, dtype=int))].reshape(shape)
                for name, off, shape in self.layout}

    def offsets(self):
        return {name: (off, shape) for name, off, shape in self.layout}

    # forward: periodic map (network.py:133-141) -> RFF (:144-147) -> tanh trunk
    # (:295-296) -> adapter tanh + PQC (:297-301) -> linear head (:302)
    def forward(self, flat, x, y, t, derivs=True):
        p = self.views(flat)
        R = len(x)
        T = self.t_domain
        raw = float(p["tau_raw"])
        tau = (1.0 + np.logaddexp(0.0, raw)) * T
        ax, ay, at = np.pi * x, np.pi * y, (t * (2.0 * np.pi)) / tau
        f = np.stack([np.sin(ax), np.cos(ax), np.sin(ay), np.cos(ay),
                      np.sin(at), np.cos(at)], axis=1)
        df = np.zeros((3, R, 6))
        df[0, :, 0], df[0, :, 1] = np.pi * np.cos(ax), -np.pi * np.sin(ax)
        df[1, :, 2], df[1, :, 3] = np.pi * np.cos(ay), -np.pi * np.sin(ay)
        w = 2.0 * np.pi / tau
        df[2, :, 4], df[2, :, 5] = w * np.cos(at), -w * np.sin(at)
        proj = f @ self.omega.T
        dproj = df @ self.omega.T
        cp, sp = np.cos(proj), np.sin(proj)
        h = np.concatenate([cp, sp], axis=1)
        dh = np.concatenate([-sp[None] * dproj, cp[None] * dproj], axis=2)
        cache = dict(x=x, y=y, t=t, tau=tau, raw=raw, at=at, f=f, df=df, proj=proj,
                     dproj=dproj, layers=[])
        for i in range(self.n_hidden):
            W, b = p[f"h{i}.W"], p[f"h{i}.b"]
            du = dh @ W
            hn = np.tanh(h @ W + b)
            cache["layers"].append((h, dh, du, hn))
            h, dh = hn, (1.0 - hn * hn)[None] * du
        if self.n_quantum:
            W, b = p["adapter.W"], p["adapter.b"]
            du = dh @ W
            a = np.tanh(h @ W + b)
            da = (1.0 - a * a)[None] * du
            cache["adapter"] = (h, dh, du, a)
            z, dz = pqc_forward(a, da, p["quantum"], self.ansatz, self.scale, self.n_layers)
            cache["pqc"] = (a, da)
            h, dh = z, dz
        out = h @ p["out.W"] + p["out.b"]
        dout = dh @ p["out.W"]
        cache["head"] = (h, dh)
        return out, dout, cache

    def backward(self, flat, cache, g_out, g_dout):
        """Reverse pass of ``forward`` given dL/d(out) [R,3] and dL/d(dout) [3,R,3]."""
        p = self.views(flat)
        off = self.offsets()
        grad = np.zeros(self.n_total)

        def put(name, g):
            o, shape = off[name]
            grad[o:o + int(np.prod(shape, dtype=int))] += np.asarray(g).ravel()

        h, dh = cache["head"]
        put("out.W", h.T @ g_out + np.einsum("kri,krj->ij", dh, g_dout))
        put("out.b", g_out.sum(axis=0))
        g_h = g_out @ p["out.W"].T
        g_dh = g_dout @ p["out.W"].T

        def tanh_lin_back(name, hin, dhin, du, y, g_y, g_dy):
            s = 1.0 - y * y
            g_u = g_y * s + np.sum(g_dy * du, axis=0) * (-2.0 * y * s)
            g_du = g_dy * s[None]
            put(f"{name}.W", hin.T @ g_u + np.einsum("kri,krj->ij", dhin, g_du))
            put(f"{name}.b", g_u.sum(axis=0))
            W = p[f"{name}.W"]
            return g_u @ W.T, g_du @ W.T

        if self.n_quantum:
            a, da = cache["pqc"]
            g_a, g_da, g_q = pqc_backward(a, da, p["quantum"], self.ansatz, self.scale,
                                          self.n_layers, g_h, g_dh)
            put("quantum", g_q)
            hin, dhin, du, y = cache["adapter"]
            g_h, g_dh = tanh_lin_back("adapter", hin, dhin, du, y, g_a, g_da)
        for i in reversed(range(self.n_hidden)):
            hin, dhin, du, y = cache["layers"][i]
            g_h, g_dh = tanh_lin_back(f"h{i}", hin, dhin, du, y, g_h, g_dh)
        # RFF: h = [cos p, sin p], dh_k = [-sin p dp_k, cos p dp_k]
        F = self.rff
        proj, dproj = cache["proj"], cache["dproj"]
        cp, sp = np.cos(proj), np.sin(proj)
        g_c, g_s = g_h[:, :F], g_h[:, F:]
        g_dc, g_ds = g_dh[:, :, :F], g_dh[:, :, F:]
        g_p = (-sp * g_c + cp * g_s
               + np.sum(-cp[None] * dproj * g_dc - sp[None] * dproj * g_ds, axis=0))
        g_dp = -sp[None] * g_dc + cp[None] * g_ds
        g_f = g_p @ self.omega
        g_df = g_dp @ self.omega
        # tau enters through at = 2 pi t / tau and df_t[4:6] = (2 pi / tau)(cos, -sin)
        tau, at = cache["tau"], cache["at"]
        ca, sa = np.cos(at), np.sin(at)
        dat = -at / tau
        w2 = 2.0 * np.pi / (tau * tau)
        g_tau = np.sum(g_f[:, 4] * ca * dat + g_f[:, 5] * (-sa) * dat
                       + g_df[2, :, 4] * (-w2 * ca + w2 * at * sa)
                       + g_df[2, :, 5] * (w2 * sa + w2 * at * ca))
        raw = cache["raw"]
        put("tau_raw", g_tau * self.t_domain * 0.5 * (1.0 + np.tanh(0.5 * raw)))
        return grad


# -- grid / loss (physics.py) ------------------------------------------------------

M_BINS = 5
IC_W = SYM_W = EN_W = 10.0  # physics.py:21-24
SYM_TERMS = {
    "vacuum": (("ez", "x", 1.0), ("ez", "y", 1.0), ("hx", "x", 1.0), ("hx", "y", -1.0),
               ("hy", "x", -1.0), ("hy", "y", 1.0)),
    "dielectric": (("ez", "y", 1.0), ("hx", "y", -1.0), ("hy", "y", 1.0)),
    "asymmetric": (),
}  # physics.py:194-205
FIELD = {"ez": 0, "hx": 1, "hy": 2}


class Grid:
    """CollocationGrid restated; physics.py:74-117."""

    def __init__(self, nx, ny, nt, t_end):
        self.nx, self.ny, self.nt, self.t_end = nx, ny, nt, t_end
        self.xs = -1.0 + 2.0 * np.arange(nx) / nx
        self.ys = -1.0 + 2.0 * np.arange(ny) / ny
        self.ts = np.linspace(0.0, t_end, nt)
        yy, xx = np.meshgrid(self.ys, self.xs, indexing="ij")
        self.x_slice, self.y_slice = xx.ravel(), yy.ravel()
        ix = np.tile(np.arange(nx), ny)
        iy = np.repeat(np.arange(ny), nx)
        self.mirror_x = iy * nx + (nx - ix) % nx
        self.mirror_y = ((ny - iy) % ny) * nx + ix
        self.s = nx * ny
        self.n_points = self.s * nt

    def bin_of_slice(self, it):
        return min(M_BINS - 1, int(self.ts[it] / (self.t_end / M_BINS)))


def time_bin_weights(bin_losses, kappa=1.0):
    """physics.py:172-180."""
    losses = np.asarray(bin_losses, dtype=np.float64)
    w = np.ones(len(losses))
    cum = 0.0
    for m in range(1, len(losses)):
        cum += losses[m - 1]
        w[m] = min(1.0, np.exp(-kappa * cum))
    return w


class Evaluator:
    """LossEvaluator restated (physics.py:263-460) with a hand-derived backward."""

    def __init__(self, model: OracleModel, grid: Grid, case="vacuum", phys_mode=None,
                 energy=True, eps_r=4.0, slab_x0=0.3, chunk_slices=4, slices=None):
        self.model, self.grid, self.case = model, grid, case
        self.phys_mode = phys_mode or ("diel_balanced" if case == "dielectric" else "vac")
        self.energy = energy
        self.eps_slice = (np.where(grid.x_slice >= slab_x0, eps_r, 1.0)
                          if case == "dielectric" else np.ones(grid.s))
        self.vac = np.flatnonzero(self.eps_slice == 1.0)
        self.diel = np.flatnonzero(self.eps_slice != 1.0)
        if case == "asymmetric":
            cx, cy, sx, sy = 0.4, 0.3, 0.85, 0.65
        else:
            cx, cy, sx, sy = 0.0, 0.0, 1.0, 1.0
        self.ic_target = np.exp(-25.0 * (((grid.x_slice - cx) / sx) ** 2
                                         + ((grid.y_slice - cy) / sy) ** 2))
        self.sym_terms = SYM_TERMS[case]
        self.bin_slices = np.array([grid.bin_of_slice(i) for i in range(grid.nt)])
        # chunks: whole slices, never straddling a bin (physics.py:305-311); ``slices``
        # restricts the sweep to a shard of time slices (data-parallel ranks)
        keep = set(range(grid.nt)) if slices is None else set(int(s) for s in slices)
        self.chunks = []
        for m in range(M_BINS):
            sl = [s for s in np.flatnonzero(self.bin_slices == m) if s in keep]
            for lo in range(0, len(sl), chunk_slices):
                sub = sl[lo:lo + chunk_slices]
                self.chunks.append((m, list(sub)))

    def _count(self, key, n_slices):
        """physics.py:432-438."""
        if key == "res1_vac":
            return n_slices * self.vac.size
        if key == "res1_diel":
            return n_slices * self.diel.size
        return n_slices * self.grid.s

    def _denom(self, key, m, weighted):
        """physics.py:440-444."""
        if weighted:
            return float(M_BINS * self._count(key, int((self.bin_slices == m).sum())))
        return float(self._count(key, self.grid.nt))

    def evaluate(self, flat, weights=None, tape=False):
        """physics.py:334-428: returns (breakdown dict, grad or None, raw sums)."""
        g, s = self.grid, self.grid.s
        N = g.n_points
        bal = self.phys_mode == "diel_balanced"
        keys = ("res1_vac", "res1_diel", "res2", "res3") if bal else ("res1", "res2", "res3")
        bin_sums = [dict() for _ in range(M_BINS)]
        sums = dict(energy=0.0, sym=0.0, ic=0.0)
        grad = np.zeros(self.model.n_total) if tape else None
        for m, sl in self.chunks:
            k = len(sl)
            x = np.tile(g.x_slice, k)
            y = np.tile(g.y_slice, k)
            t = np.repeat(g.ts[sl], s)
            eps = np.tile(self.eps_slice, k)
            out, dout, cache = self.model.forward(flat, x, y, t)
            ez, hx, hy = out[:, 0], out[:, 1], out[:, 2]
            ezx, ezy, ezt = dout[0, :, 0], dout[1, :, 0], dout[2, :, 0]
            hxx, hxy, hxt = dout[0, :, 1], dout[1, :, 1], dout[2, :, 1]
            hyx, hyy, hyt = dout[0, :, 2], dout[1, :, 2], dout[2, :, 2]
            res1 = ezt - (hyx - hxy) / eps
            res2 = hxt + ezy
            res3 = hyt - ezx
            g_out = np.zeros_like(out)
            g_dout = np.zeros_like(dout)
            w_m = 1.0 if weights is None else float(weights[m])
            c1 = np.zeros_like(res1)
            if bal:
                vi = (np.arange(k)[:, None] * s + self.vac[None]).ravel()
                di = (np.arange(k)[:, None] * s + self.diel[None]).ravel()
                parts = [("res1_vac", np.sum(res1[vi] ** 2)), ("res1_diel", np.sum(res1[di] ** 2))]
                c1[vi] = w_m / self._denom("res1_vac", m, weights is not None)
                c1[di] = w_m / self._denom("res1_diel", m, weights is not None)
            else:
                parts = [("res1", np.sum(res1 ** 2))]
                c1[:] = w_m / self._denom("res1", m, weights is not None)
            parts += [("res2", np.sum(res2 ** 2)), ("res3", np.sum(res3 ** 2))]
            c2 = w_m / self._denom("res2", m, weights is not None)
            c3 = w_m / self._denom("res3", m, weights is not None)
            for key, v in parts:
                bin_sums[m][key] = bin_sums[m].get(key, 0.0) + float(v)
            # d/d(derivs) of the residual terms
            g_dout[2, :, 0] += 2 * c1 * res1
            g_dout[0, :, 2] += -2 * c1 * res1 / eps
            g_dout[1, :, 1] += 2 * c1 * res1 / eps
            g_dout[2, :, 1] += 2 * c2 * res2
            g_dout[1, :, 0] += 2 * c2 * res2
            g_dout[2, :, 2] += 2 * c3 * res3
            g_dout[0, :, 0] += -2 * c3 * res3
            if self.energy:
                rE = (eps * ez * ezt + hx * hxt + hy * hyt) - (ezx * hy + ez * hyx) \
                    + (ezy * hx + ez * hxy)  # physics.py:157-164
                sums["energy"] += float(np.sum(rE * rE))
                gE = 2.0 * (EN_W / N) * rE
                g_out[:, 0] += gE * (eps * ezt - hyx + hxy)
                g_out[:, 1] += gE * (hxt + ezy)
                g_out[:, 2] += gE * (hyt - ezx)
                g_dout[2, :, 0] += gE * eps * ez
                g_dout[2, :, 1] += gE * hx
                g_dout[2, :, 2] += gE * hy
                g_dout[0, :, 0] += gE * (-hy)
                g_dout[0, :, 2] += gE * (-ez)
                g_dout[1, :, 0] += gE * hx
                g_dout[1, :, 1] += gE * ez
            if self.sym_terms:
                offs = (np.arange(k) * s)[:, None]
                mx = (offs + g.mirror_x[None]).ravel()
                my = (offs + g.mirror_y[None]).ravel()
                for name, axis, sign in self.sym_terms:
                    fi = FIELD[name]
                    f = out[:, fi]
                    mir = f[mx if axis == "x" else my]
                    d = f - sign * mir
                    sums["sym"] += float(np.sum(d * d))
                    g_out[:, fi] += (SYM_W / N) * 4.0 * d
            if sl[0] == 0:
                dz = ez[:s] - self.ic_target
                sums["ic"] += float(np.sum(dz * dz) + np.sum(hx[:s] ** 2) + np.sum(hy[:s] ** 2))
                cI = 2.0 * IC_W / s
                g_out[:s, 0] += cI * dz
                g_out[:s, 1] += cI * hx[:s]
                g_out[:s, 2] += cI * hy[:s]
            if tape:
                grad += self.model.backward(flat, cache, g_out, g_dout)
        return self._breakdown(bin_sums, sums, weights), grad, (bin_sums, sums)

    def _bin_loss(self, m, d):
        """physics.py:446-450."""
        n_sl = int((self.bin_slices == m).sum())
        if n_sl == 0:
            return 0.0
        return sum(v / self._count(k, n_sl) for k, v in d.items())

    def _breakdown(self, bin_sums, sums, weights):
        """physics.py:416-426."""
        g = self.grid
        bin_phys = tuple(self._bin_loss(m, bin_sums[m]) for m in range(M_BINS))
        if weights is None:
            keys = set()
            for d in bin_sums:
                keys.update(d)
            phys = sum(sum(d.get(k, 0.0) for d in bin_sums) / self._count(k, g.nt)
                       for k in keys)
        else:
            phys = float(np.mean([weights[m] * bin_phys[m] for m in range(M_BINS)]))
        ic = sums["ic"] / g.s
        sym = sums["sym"] / g.n_points
        energy = sums["energy"] / g.n_points if self.energy else 0.0
        total = phys + IC_W * ic + SYM_W * sym + (EN_W * energy if self.energy else 0.0)
        return dict(phys=phys, ic=ic, sym=sym, energy=energy, total=total,
                    bin_phys=bin_phys)


# -- trainer (training.py) ----------------------------------------------------------

def lr_at(epoch, lr0=1e-3, decay=0.85, every=2000):
    """training.py:82-84."""
    return lr0 * decay ** (epoch // every)


def init_quantum_params(strategy, count, seed=0):
    """training.py:69-79."""
    if strategy == "reg":
        return np.random.default_rng(seed).uniform(0.0, 2.0 * np.pi, count)
    return np.full(count, {"zeros": 0.0, "pi": np.pi, "pi_half": np.pi / 2.0}[strategy])


def adam_update(flat, grad, m, v, t, lr, b1=0.9, b2=0.999, eps=1e-8):
    """training.py:101-111 (in place on flat, m, v); returns new t."""
    if not np.all(np.isfinite(grad)):
        raise OracleError("non-finite gradient")
    t += 1
    m[:] = b1 * m + (1.0 - b1) * grad
    v[:] = b2 * v + (1.0 - b2) * grad * grad
    mhat = m / (1.0 - b1 ** t)
    vhat = v / (1.0 - b2 ** t)
    flat -= lr * mhat / (np.sqrt(vhat) + eps)
    return t


def train_curve(model: OracleModel, grid: Grid, epochs, case="vacuum", energy=True,
                phys_mode=None, seed=0, init_strategy="reg", adaptive=True, kappa=1.0,
                chunk_slices=4, lr0=1e-3):
    """training.py:309-414 without probes: per-epoch breakdowns and final params."""
    flat = model.init_params()
    if model.n_quantum:
        flat[model.n_classical:] = init_quantum_params(init_strategy, model.n_quantum, seed)
    ev = Evaluator(model, grid, case=case, phys_mode=phys_mode, energy=energy,
                   chunk_slices=chunk_slices)
    weights = None
    if adaptive:
        weights = time_bin_weights(ev.evaluate(flat)[0]["bin_phys"], kappa)
    m = np.zeros(model.n_total)
    v = np.zeros(model.n_total)
    t = 0
    rows = []
    for epoch in range(epochs):
        bd, grad, _ = ev.evaluate(flat, weights, tape=True)
        rows.append(bd)
        t = adam_update(flat, grad, m, v, t, lr_at(epoch, lr0))
        if adaptive:
            weights = time_bin_weights(bd["bin_phys"], kappa)
    return rows, flat


# ---- diagnostic probes -------------------------------------------------
def pqc_state(a, qp, kind, scale, n_layers):
    """Final circuit state psi [R, 2^n] for value-only inputs (the state the
    Meyer-Wallach probe reads); ansatz.py:215-227 via the fused plan."""
    a = np.asarray(a, dtype=np.float64)
    R, n = a.shape
    gates, _ = build_circuit(kind, n, n_layers)
    theta, _, _ = scale_derivs(scale, a)
    return _run_steps(_product_state(theta, n), n, fused_plan(gates, n), qp)


def meyer_wallach(psi):
    """Q = 2 (1 - mean_k Tr rho_k^2) per row; qsim.py:384-406."""
    psi = np.atleast_2d(psi)
    R, D = psi.shape
    n = int(round(math.log2(D)))
    pur = np.zeros(R)
    for k in range(n):
        v = psi.reshape(R, 2 ** k, 2, 2 ** (n - k - 1))
        v = np.moveaxis(v, 2, 1).reshape(R, 2, -1)
        rho = v @ np.conj(np.swapaxes(v, 1, 2))
        pur += np.sum(rho.real ** 2 + rho.imag ** 2, axis=(1, 2))
    return 2.0 * (1.0 - pur / n)


def model_predict(model: "OracleModel", flat, x, y, t):
    """Value-only fields (E_z, H_x, H_y) [3, R]; network.py:310-321."""
    out, _, _ = model.forward(flat, np.asarray(x, float), np.asarray(y, float),
                              np.asarray(t, float))
    return out.T


def adapter_activations(model: "OracleModel", flat, x, y, t):
    """Pre-embedding activations a [R, n]; network.py:323-335."""
    _, _, cache = model.forward(flat, np.asarray(x, float), np.asarray(y, float),
                                np.asarray(t, float))
    return cache["pqc"][0]


def probe_entanglement(model: "OracleModel", flat, x, y, t):
    """Mean Meyer-Wallach Q at the probe inputs; training.py:174-184."""
    a = adapter_activations(model, flat, x, y, t)
    qp = model.views(flat)["quantum"]
    return float(np.mean(meyer_wallach(pqc_state(a, qp, model.ansatz, model.scale,
                                                  model.n_layers))))


def epsilon_at(case, x, eps_r=4.0, slab_x0=0.3):
    """physics.py:45-49."""
    x = np.asarray(x, dtype=np.float64)
    if case != "dielectric":
        return np.ones_like(x)
    return np.where(x >= slab_x0, eps_r, 1.0)


def total_energy(ez, hx, hy, eps, dx, dy):
    """0.5 Riemann sum of eps Ez^2 + Hx^2 + Hy^2; fdtd.py:194-197."""
    return float(np.sum(0.5 * (eps * ez * ez + hx * hx + hy * hy)) * dx * dy)


def energy_probe(model: "OracleModel", flat, case, nx, ny, times):
    """U_theta(t_k) on the collocated nx x ny grid; training.py:187-200."""
    xs = -1.0 + 2.0 * np.arange(nx) / nx
    ys = -1.0 + 2.0 * np.arange(ny) / ny
    yy, xx = np.meshgrid(ys, xs, indexing="ij")
    xf, yf = xx.ravel(), yy.ravel()
    eps = epsilon_at(case, xf)
    out = np.zeros(len(times))
    for k, tk in enumerate(times):
        ez, hx, hy = model_predict(model, flat, xf, yf, np.full_like(xf, tk))
        out[k] = total_energy(ez, hx, hy, eps, 2.0 / nx, 2.0 / ny)
    return out


def bh_index(u, times=None):
    """(clamped, raw) 1 - min_{t > 0} U(t)/U(0); training.py:117-134."""
    u = np.asarray(u, dtype=np.float64)
    if u[0] <= 0.0:
        raise OracleError("U(0) must be positive")
    mask = (np.asarray(times) > 0.0) if times is not None else (np.arange(len(u)) > 0)
    raw = 1.0 - float(np.min((u / u[0])[mask]))
    return float(np.clip(raw, 0.0, 1.0)), raw


def l2_against_reference(model: "OracleModel", flat, times, xs, ys, ez_ref):
    """Relative L2 of E_z on the snapshot grid; training.py:203-217."""
    yy, xx = np.meshgrid(ys, xs, indexing="ij")
    xf, yf = xx.ravel(), yy.ravel()
    num = den = 0.0
    for k, tk in enumerate(times):
        ez = model_predict(model, flat, xf, yf, np.full_like(xf, tk))[0]
        ref = ez_ref[k].ravel()
        num += float(np.sum((ez - ref) ** 2))
        den += float(np.sum(ref * ref))
    return float(np.sqrt(num / den))


# ---- FDTD reference solver ---------------------------------------------
def fdtd_run(nx, ny, case="vacuum", t_end=1.5, cfl=0.5, ic="pulse", n_snapshots=100,
             eps_r=4.0, slab_x0=0.3, center=(0.0, 0.0), stretch=(1.0, 1.0)):
    """Yee TEz leapfrog on the periodic cell with collocated snapshots;
    fdtd.py:115-181 (H at t = -dt/2 from a discrete half step, Ez update with
    a pointwise epsilon, snapshots at the steps nearest linspace(0, t_end))."""
    dx, dy = 2.0 / nx, 2.0 / ny
    dt0 = cfl * min(dx, dy) / np.sqrt(2.0)
    steps = max(1, int(np.ceil(t_end / dt0 - 1e-12)))
    dt = t_end / steps
    xs = -1.0 + dx * np.arange(nx)
    ys = -1.0 + dy * np.arange(ny)
    yy, xx = np.meshgrid(ys, xs, indexing="ij")
    eps = epsilon_at(case, xx, eps_r, slab_x0)
    if ic == "plane_wave":
        ez = np.cos(np.pi * xx)
        hx = np.zeros_like(ez)
        hy = np.cos(np.pi * (xx + dx / 2.0 - dt / 2.0))
    else:
        ez = np.exp(-25.0 * (((xx - center[0]) / stretch[0]) ** 2
                             + ((yy - center[1]) / stretch[1]) ** 2))
        hx = (dt / 2.0) * (np.roll(ez, -1, axis=0) - ez) / dy
        hy = -(dt / 2.0) * (np.roll(ez, -1, axis=1) - ez) / dx
    wanted = np.linspace(0.0, t_end, n_snapshots)
    snap = set(int(s) for s in np.unique(np.clip(np.round(wanted / dt).astype(int), 0, steps)))
    times, rez, rhx, rhy = [], [], [], []
    for step in range(steps + 1):
        hx_new = hx - (dt / dy) * (np.roll(ez, -1, axis=0) - ez)
        hy_new = hy + (dt / dx) * (np.roll(ez, -1, axis=1) - ez)
        if step in snap:
            hxm, hym = 0.5 * (hx + hx_new), 0.5 * (hy + hy_new)
            times.append(step * dt)
            rez.append(ez.copy())
            rhx.append(0.5 * (hxm + np.roll(hxm, 1, axis=0)))
            rhy.append(0.5 * (hym + np.roll(hym, 1, axis=1)))
        hx, hy = hx_new, hy_new
        ez = ez + (dt / eps) * ((hy - np.roll(hy, 1, axis=1)) / dx
                                - (hx - np.roll(hx, 1, axis=0)) / dy)
    return dict(times=np.array(times), ez=np.stack(rez), hx=np.stack(rhx), hy=np.stack(rhy),
                xs=xs, ys=ys, dt=dt, steps=steps, eps=eps)
