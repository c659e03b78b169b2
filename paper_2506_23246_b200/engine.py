"""Native epoch sweep for hybrid QPINN models: every kernel of the step is ours.

One chunk of whole time slices runs (network.py:284-308, physics.py:352-414):

    qpinn_trunk_forward          periodic map + RFF + tanh layers + adapter, with x/y/t tangents
    qpinn_pqc_forward     (K1)   scaled embedding -> PQC -> <Z>, tangents, state hand-off
    qpinn_loss_head_...   (K4)   linear head + residuals + every loss term + dL/dz, dL/dhead
    qpinn_pqc_backward    (K2)   adjoint: dL/d(act, act tangents), dL/dqparams
    qpinn_trunk_backward         dL/d(trunk weights, biases, tau_raw)

There is no autograd graph: the engine calls the C ABI in order on the
current stream, with all buffers preallocated per chunk, so a whole epoch
is a fixed launch sequence (CUDA-graph capturable).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np
import torch

from . import _native as N
from .ansatz import _SCALE_CODE, ScaleKind, state_buffer


def adapter_fused(model) -> bool:
    """trunk.cu's rule: the float32 dual forward computes the tanh adapter in the
    last hidden layer's tensor-core epilogue (QPINN_FUSE_ADAPTER=0 turns it off)."""
    import os
    cfg = model.config
    H = cfg.hidden_width
    return (model.dtype == torch.float32 and model.n_hidden > 0 and H <= 128 and H % 4 == 0
            and cfg.n_qubits <= 8 and os.environ.get("QPINN_FUSE_ADAPTER", "1") != "0")


def trunk_desc(model):
    """``qpinn_trunk_desc`` for a hybrid model (offsets into its flat layout);
    returns (desc, omega tensor kept alive, offsets)."""
    cfg = model.config
    off = {name: o for name, o, _ in model.layout}
    d = N.TrunkDesc()
    d.n_hidden = model.n_hidden
    d.rff = cfg.rff_features
    d.hidden = cfg.hidden_width
    d.n_out = cfg.n_qubits
    for i in range(model.n_hidden):
        d.off_w[i] = off[f"h{i}.W"]
        d.off_b[i] = off[f"h{i}.b"]
    d.off_adapter_w = off["adapter.W"]
    d.off_adapter_b = off["adapter.b"]
    d.off_tau_raw = off["tau_raw"]
    d.t_domain = cfg.t_domain
    omega = model.omega.contiguous()
    d.omega = omega.data_ptr()
    return d, omega, off


class InferenceEngine:
    """Value-only evaluation of a hybrid model with our kernels only
    (network.py:310-335): value trunk (tensor-core dense layers with the tanh
    epilogue) -> K1 without tangents -> linear head, in fixed chunks.  Also
    the Meyer-Wallach probe (K1 with the per-qubit coherence readout)."""

    def __init__(self, model, chunk: int = 1 << 16):
        if model.circuit is None:
            raise ValueError("the inference engine needs a hybrid model")
        self.model = model
        self.chunk = chunk
        cfg = model.config
        self.n = cfg.n_qubits
        self.device, self.dtype = model.device, model.dtype
        self.dcode = N.dtype_code(self.dtype)
        self.scale = _SCALE_CODE[ScaleKind(cfg.scale)]
        self.desc, self._omega, off = trunk_desc(model)
        self.off_out_w, self.off_out_b, self.off_q = off["out.W"], off["out.b"], off["quantum"]
        lib = N.lib()
        dev, dt, n = self.device, self.dtype, self.n
        self.trunk_ws = torch.empty(lib.qpinn_trunk_workspace_bytes(C.byref(self.desc),
                                                                    self.dcode, chunk),
                                    dtype=torch.uint8, device=dev)
        # private scratch: the running |a| maximum must not mix with training's
        self.pqc_ws = torch.zeros(lib.qpinn_pqc_workspace_bytes(model.circuit.handle, self.dcode,
                                                                chunk),
                                  dtype=torch.uint8, device=dev)
        self.act = torch.empty((chunk, n), dtype=dt, device=dev)
        self.z = torch.empty((chunk, n), dtype=dt, device=dev)
        self.coh = torch.empty((chunk, n, 2), dtype=dt, device=dev)

    def _chunks(self, x):
        for lo in range(0, x.shape[0], self.chunk):
            yield lo, min(x.shape[0], lo + self.chunk)

    def _trunk_pqc(self, flat, x, y, t, lo, hi, probe):
        lib, st, es, dc = N.lib(), N.stream_ptr(), flat.element_size(), self.dcode
        R = hi - lo
        fp = flat.data_ptr()
        N.check(lib.qpinn_trunk_forward_value(
            C.byref(self.desc), dc, R, x[lo:].data_ptr(), y[lo:].data_ptr(), t[lo:].data_ptr(),
            fp, self.act.data_ptr(), self.trunk_ws.data_ptr(), self.trunk_ws.numel(), st),
            "qpinn_trunk_forward_value")
        qp = fp + self.off_q * es
        if probe:
            N.check(lib.qpinn_pqc_forward_probe(
                self.model.circuit.handle, dc, self.scale, R, self.act.data_ptr(), qp,
                self.z.data_ptr(), self.coh.data_ptr(), self.pqc_ws.data_ptr(),
                self.pqc_ws.numel(), st), "qpinn_pqc_forward_probe")
        else:
            N.check(lib.qpinn_pqc_forward(
                self.model.circuit.handle, dc, self.scale, R, self.act.data_ptr(), 0, qp,
                self.z.data_ptr(), 0, 0, self.pqc_ws.data_ptr(), self.pqc_ws.numel(), st),
                "qpinn_pqc_forward")
        widths = [2 * self.model.config.rff_features] + \
            [self.model.config.hidden_width] * self.model.n_hidden
        N.count_launches(1 + sum(2 if (self.dtype == torch.float32 and k % 4 == 0) else 1
                                 for k in widths) + 2)

    def _trunk_launches(self, dual: bool = False) -> int:
        widths = [2 * self.model.config.rff_features] + \
            [self.model.config.hidden_width] * self.model.n_hidden
        n = 1 + sum(2 if (self.dtype == torch.float32 and k % 4 == 0) else 1 for k in widths)
        return n - 2 if dual and adapter_fused(self.model) else n

    def adapter(self, flat, x, y, t) -> torch.Tensor:
        """Adapter activations a [R, n] (network.py:323-335): value trunk only."""
        lib, st, dc = N.lib(), N.stream_ptr(), self.dcode
        R = x.shape[0]
        out = torch.empty((R, self.n), dtype=self.dtype, device=self.device)
        for lo, hi in self._chunks(x):
            N.check(lib.qpinn_trunk_forward_value(
                C.byref(self.desc), dc, hi - lo, x[lo:].data_ptr(), y[lo:].data_ptr(),
                t[lo:].data_ptr(), flat.data_ptr(), out[lo:].data_ptr(), self.trunk_ws.data_ptr(),
                self.trunk_ws.numel(), st), "qpinn_trunk_forward_value")
            N.count_launches(self._trunk_launches())
        return out

    def dual_fields(self, flat, x, y, t):
        """(out [R, 3], dout [3, R, 3]): fields and their x/y/t jacobians
        (network.py:284-308 with derivs) on our kernels only: the dual trunk
        (tensor-core layers with the fused dual tanh), K1 with tangents, the
        head kernel on the values and on the stacked tangents."""
        lib, st, dc, n = N.lib(), N.stream_ptr(), self.dcode, self.n
        es = flat.element_size()
        R = x.shape[0]
        if getattr(self, "_act4", None) is None:
            self._act4 = torch.empty(4 * self.chunk * n, dtype=self.dtype, device=self.device)
            self._z4 = torch.empty(4 * self.chunk * n, dtype=self.dtype, device=self.device)
            self._dout = torch.empty(3 * self.chunk * 3, dtype=self.dtype, device=self.device)
            self._zero_b = torch.zeros(3, dtype=self.dtype, device=self.device)
        out = torch.empty((R, 3), dtype=self.dtype, device=self.device)
        dout = torch.empty((3, R, 3), dtype=self.dtype, device=self.device)
        fp = flat.data_ptr()
        w_out, b_out = fp + self.off_out_w * es, fp + self.off_out_b * es
        for lo, hi in self._chunks(x):
            r = hi - lo
            a0, z0 = self._act4.data_ptr(), self._z4.data_ptr()
            N.check(lib.qpinn_trunk_forward(
                C.byref(self.desc), dc, r, x[lo:].data_ptr(), y[lo:].data_ptr(),
                t[lo:].data_ptr(), fp, a0, self.trunk_ws.data_ptr(), self.trunk_ws.numel(), st),
                "qpinn_trunk_forward")
            N.check(lib.qpinn_pqc_forward(
                self.model.circuit.handle, dc, self.scale, r, a0, a0 + r * n * es,
                fp + self.off_q * es, z0, z0 + r * n * es, 0, self.pqc_ws.data_ptr(),
                self.pqc_ws.numel(), st), "qpinn_pqc_forward")
            N.check(lib.qpinn_head_forward(dc, r, n, z0, w_out, b_out, out[lo:].data_ptr(), st),
                    "qpinn_head_forward")
            N.check(lib.qpinn_head_forward(dc, 3 * r, n, z0 + r * n * es, w_out,
                                           self._zero_b.data_ptr(), self._dout.data_ptr(), st),
                    "qpinn_head_forward")
            dout[:, lo:hi].copy_(self._dout[:3 * r * 3].view(3, r, 3))
            N.count_launches(self._trunk_launches(dual=True) + 2 + 2)
        return out, dout

    def check_domain(self):
        """The reference's |a| <= 1 rule on every forward since the last check."""
        from .ansatz import check_domain
        return check_domain(self.model.circuit, self.dtype, self.device, ws=self.pqc_ws)

    def fields(self, flat, x, y, t, out=None):
        """(E_z, H_x, H_y) as a [R, 3] device tensor."""
        lib, st = N.lib(), N.stream_ptr()
        es = flat.element_size()
        R = x.shape[0]
        out = torch.empty((R, 3), dtype=self.dtype, device=self.device) if out is None else out
        for lo, hi in self._chunks(x):
            self._trunk_pqc(flat, x, y, t, lo, hi, False)
            N.check(lib.qpinn_head_forward(self.dcode, hi - lo, self.n, self.z.data_ptr(),
                                           flat.data_ptr() + self.off_out_w * es,
                                           flat.data_ptr() + self.off_out_b * es,
                                           out[lo:].data_ptr(), st), "qpinn_head_forward")
            N.count_launches(1)
        return out

    def meyer_wallach(self, flat, x, y, t):
        """Per-point Meyer-Wallach Q (qsim.py:384-406) of the circuit state."""
        R = x.shape[0]
        q = torch.empty(R, dtype=torch.float64, device=self.device)
        for lo, hi in self._chunks(x):
            self._trunk_pqc(flat, x, y, t, lo, hi, True)
            z = self.z[:hi - lo].double()
            c = self.coh[:hi - lo].double()
            purity = 0.5 * (1.0 + z * z) + 2.0 * (c[..., 0] ** 2 + c[..., 1] ** 2)
            q[lo:hi] = 2.0 * (1.0 - purity.mean(dim=1))
        return q


class _ChunkBuffers:
    def __init__(self, engine, ch):
        R = ch.x.numel()
        n, dev, dt = engine.n, engine.device, engine.dtype
        self.R = R
        self.act = torch.empty((4, R, n), dtype=dt, device=dev)
        self.z = torch.empty((4, R, n), dtype=dt, device=dev)
        self.gz = torch.empty((4, R, n), dtype=dt, device=dev)
        self.gact = torch.empty((4, R, n), dtype=dt, device=dev)
        self.states = state_buffer(engine.circuit, self.act[0])
        self.sums = torch.zeros(N.LOSS_NSUMS, dtype=torch.float64, device=dev)


class NativeEngine:
    """Preallocated native trunk -> K1 -> K4 -> K2 -> trunk^T sweep."""

    def __init__(self, model, evaluator):
        if model.circuit is None:
            raise ValueError("the native engine needs a hybrid model")
        cfg = model.config
        self.model, self.ev = model, evaluator
        self.circuit = model.circuit
        self.n = cfg.n_qubits
        self.device, self.dtype = model.device, model.dtype
        self.dcode = N.dtype_code(self.dtype)
        self.scale = _SCALE_CODE[ScaleKind(cfg.scale)]
        self.desc, self._omega, off = trunk_desc(model)
        self.off_out_w, self.off_out_b = off["out.W"], off["out.b"]
        self.off_q = off["quantum"]
        lib = N.lib()
        self.chunks = evaluator.chunks
        self.bufs: List[_ChunkBuffers] = [_ChunkBuffers(self, ch) for ch in self.chunks]
        rmax = max((b.R for b in self.bufs), default=0)
        self.trunk_ws = torch.empty(lib.qpinn_trunk_workspace_bytes(C.byref(self.desc),
                                                                    self.dcode, rmax),
                                    dtype=torch.uint8, device=self.device)
        self.loss_ws = torch.empty(lib.qpinn_loss_workspace_bytes(None, 0, 0), dtype=torch.uint8,
                                   device=self.device)
        self.pqc_ws = self.circuit.workspace(self.dtype, self.device, rmax)
        self._has_phase = any(s[0] == "phases" for s in self.circuit.fused_plan())
        self.grad_chunk = (torch.empty(model.total_parameter_count, dtype=self.dtype,
                                       device=self.device) if len(self.chunks) > 1 else None)

    def sweep(self, flat: torch.Tensor, grad: Optional[torch.Tensor], weights_dev,
              sums_out: torch.Tensor, tape: bool = True) -> None:
        """Forward (+ full gradient into ``grad`` when tape) over every chunk;
        raw loss sums accumulate into ``sums_out`` (float64 [23]; with one chunk they
        overwrite it)."""
        lib = N.lib()
        st = N.stream_ptr()
        fp = flat.data_ptr()
        dc, n = self.dcode, self.n
        es = flat.element_size()
        wptr = N.ptr(weights_dev)
        # one chunk: the loss reduction writes (not adds) the sums straight into sums_out
        direct = len(self.chunks) == 1 and sums_out.is_contiguous()
        for i, (ch, b) in enumerate(zip(self.chunks, self.bufs)):
            R = b.R
            g = grad if (self.grad_chunk is None or grad is None) else self.grad_chunk
            gp = g.data_ptr() if g is not None else 0
            with N.timed("trunk_forward"):
                N.check(lib.qpinn_trunk_forward(C.byref(self.desc), dc, R, ch.x.data_ptr(),
                                                ch.y.data_ptr(), ch.t.data_ptr(), fp,
                                                b.act.data_ptr(), self.trunk_ws.data_ptr(),
                                                self.trunk_ws.numel(), st), "qpinn_trunk_forward")
            a0 = b.act.data_ptr()
            a1 = a0 + R * n * es
            with N.timed("pqc_forward"):
                N.check(lib.qpinn_pqc_forward(self.circuit.handle, dc, self.scale, R, a0, a1,
                                              fp + self.off_q * es, b.z.data_ptr(),
                                              b.z.data_ptr() + R * n * es,
                                              b.states.data_ptr() if tape else 0,
                                              self.pqc_ws.data_ptr(), self.pqc_ws.numel(), st),
                        "qpinn_pqc_forward")
            scratch_w = g if g is not None else b.gact  # dL/dhead lands in grad (or scratch)
            with N.timed("loss"):
                N.check(lib.qpinn_loss_head_forward_backward(
                    C.byref(ch.spec), dc, R, n, b.z.data_ptr(), fp + self.off_out_w * es,
                    fp + self.off_out_b * es, wptr, b.gz.data_ptr(),
                    (gp + self.off_out_w * es) if g is not None else scratch_w.data_ptr(),
                    (gp + self.off_out_b * es) if g is not None else scratch_w.data_ptr() + 64 * es,
                    (sums_out if direct else b.sums).data_ptr(), self.loss_ws.data_ptr(),
                    self.loss_ws.numel(), st),
                    "qpinn_loss_head_forward_backward")
            if tape:
                gz0 = b.gz.data_ptr()
                ga0 = b.gact.data_ptr()
                with N.timed("pqc_backward"):
                    N.check(lib.qpinn_pqc_backward(
                        self.circuit.handle, dc, self.scale, R, a0, a1, fp + self.off_q * es,
                        b.states.data_ptr(), gz0, gz0 + R * n * es, ga0, ga0 + R * n * es,
                        gp + self.off_q * es, self.pqc_ws.data_ptr(), self.pqc_ws.numel(), st),
                        "qpinn_pqc_backward")
                with N.timed("trunk_backward"):
                    N.check(lib.qpinn_trunk_backward(C.byref(self.desc), dc, R, ch.x.data_ptr(),
                                                     ch.y.data_ptr(), ch.t.data_ptr(), fp, a0,
                                                     ga0, gp, self.trunk_ws.data_ptr(),
                                                     self.trunk_ws.numel(), st),
                            "qpinn_trunk_backward")
                if g is not grad:
                    if i == 0:
                        grad.copy_(g)
                    else:
                        grad.add_(g)
            if not direct:
                sums_out += b.sums
            N.count_launches(self._launches(tape))

    def _launches(self, tape: bool) -> int:
        """Our kernels per chunk (cuBLAS GEMMs excluded), mirroring trunk.cu's
        per-layer choice: float32 layers with 16-byte aligned widths run on the
        tensor-core kernels (weight split + GEMM with fused dual tanh), the rest
        on cuBLAS + a separate dual-tanh kernel."""
        cfg = self.model.config
        f32 = self.dtype == torch.float32
        widths = [2 * cfg.rff_features] + [cfg.hidden_width] * self.model.n_hidden
        phase = 1 if self._has_phase else 0
        n = 1                                   # features
        for k in widths:                        # hidden layers + adapter (input width k)
            n += 2 if (f32 and k % 4 == 0) else 1
        if adapter_fused(self.model):           # the adapter rides in the last layer's epilogue
            n -= 2
        n += 2 + 2                              # K1 prep + main, K4 + reduce
        if tape:
            n += 4 + phase                      # K2 prep, main, reduce, u1 grads (+ phase grads)
            H = cfg.hidden_width
            fused = self.model.n_hidden > 0 and self.n <= 16 and H <= 128
            # adapter: fused with the last hidden layer's reverse tanh (kernel + 3 reduces),
            # else reverse dual tanh + bias reduce (its GEMMs are cuBLAS)
            n += 4 if fused else 2
            for li, k in enumerate(widths[:-1] if self.model.n_hidden else []):
                if not (fused and li == self.model.n_hidden - 1):
                    n += 2 if H <= 256 else 3   # reverse dual tanh (+ fused bias partials), reduce
                if f32 and k % 4 == 0 and H % 4 == 0:
                    n += 2                      # weight gradient: split-K kernel + reduce
                if f32 and H % 4 == 0:
                    n += 2                      # input gradient: weight split + GEMM
            n += 2                              # tau: features_bwd + reduce
        return n
