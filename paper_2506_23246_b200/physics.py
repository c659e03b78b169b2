"""Residuals, loss terms and the fused epoch evaluator on the device.

Mirrors ``qpinn.physics`` (physics.py): ``MaterialMap`` (:30-49),
``PulseSpec`` (:52-67), ``CollocationGrid`` (:74-117), ``time_bin_weights``
(:172-180), ``total_loss`` (:183-187), the parity term tables (:194-205) and
``LossEvaluator`` (:263-460).  Every static table (coordinates, permittivity,
pulse, time bins, region counts) is derived on the host with the reference's
own numpy expressions, then kept resident on the device; the per-point
residual/loss/gradient work runs in the fused K4 kernel and the breakdown and
next adaptive weights are finalised on the device.

Data-parallel sharding: an evaluator built with ``slices=`` covers a subset of
whole time slices; every coefficient keeps its *global* normalisation, so the
sum over shards of gradients and raw sums is exactly the full-grid result
(SURVEY 8e).  ``reduce_fn`` (e.g. an NCCL all-reduce) combines the packed
[grad, sums] vector before finalisation.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError
from .network import FieldBatch, FieldDerivs, Model, ParameterStore

M_BINS = 5
IC_WEIGHT = 10.0
SYM_WEIGHT = 10.0
ENERGY_WEIGHT = 10.0
CASES = ("vacuum", "dielectric", "asymmetric")
PHYS_MODES = ("vac", "diel_balanced", "intuitive")
KEYS_VAC = ("res1", "res2", "res3")
KEYS_BAL = ("res1_vac", "res1_diel", "res2", "res3")
_KEY_SLOT = {"res1": 0, "res1_vac": 0, "res1_diel": 1, "res2": 2, "res3": 3}


@dataclass(frozen=True)
class MaterialMap:
    """Pointwise relative permittivity; slab x >= slab_x0 in the dielectric case."""
    case: str = "vacuum"
    eps_r: float = 4.0
    slab_x0: float = 0.3

    def __post_init__(self):
        if self.case not in CASES:
            raise ConfigError(f"unknown case {self.case!r}")

    def epsilon_at(self, x, y) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        if self.case != "dielectric":
            return np.ones_like(x)
        return np.where(x >= self.slab_x0, self.eps_r, 1.0)


@dataclass(frozen=True)
class PulseSpec:
    """Gaussian initial pulse exp(-25 [((x-cx)/sx)^2 + ((y-cy)/sy)^2])."""
    center: tuple = (0.0, 0.0)
    stretch: tuple = (1.0, 1.0)

    @classmethod
    def for_case(cls, case: str) -> "PulseSpec":
        if case == "asymmetric":
            return cls(center=(0.4, 0.3), stretch=(0.85, 0.65))
        return cls()

    def ez0(self, x, y) -> np.ndarray:
        cx, cy = self.center
        sx, sy = self.stretch
        return np.exp(-25.0 * (((x - cx) / sx) ** 2 + ((y - cy) / sy) ** 2))


def default_t_end(case: str) -> float:
    return 0.7 if case == "dielectric" else 1.5


@dataclass
class CollocationGrid:
    """Uniform (x, y, t) grid, t-major then y then x (physics.py:74-117)."""
    nx: int
    ny: int
    nt: int
    t_end: float

    def __post_init__(self):
        self.xs = -1.0 + 2.0 * np.arange(self.nx) / self.nx
        self.ys = -1.0 + 2.0 * np.arange(self.ny) / self.ny
        self.ts = np.linspace(0.0, self.t_end, self.nt)
        yy, xx = np.meshgrid(self.ys, self.xs, indexing="ij")
        self.x_slice = xx.ravel()
        self.y_slice = yy.ravel()
        ix = np.tile(np.arange(self.nx), self.ny)
        iy = np.repeat(np.arange(self.ny), self.nx)
        self.mirror_x_local = iy * self.nx + (self.nx - ix) % self.nx
        self.mirror_y_local = ((self.ny - iy) % self.ny) * self.nx + ix

    @property
    def slice_size(self) -> int:
        return self.nx * self.ny

    @property
    def n_points(self) -> int:
        return self.slice_size * self.nt

    def flat_points(self):
        s = self.slice_size
        return (np.tile(self.x_slice, self.nt), np.tile(self.y_slice, self.nt),
                np.repeat(self.ts, s))

    def bin_of_slice(self, it: int) -> int:
        edge = self.t_end / M_BINS
        return min(M_BINS - 1, int(self.ts[it] / edge))


# -- pointwise physics (tensor utilities, physics.py:123-187) --------------------

def pde_residuals(fields: FieldBatch, derivs: FieldDerivs, eps):
    res1 = derivs.ez_t - (derivs.hy_x - derivs.hx_y) / eps
    res2 = derivs.hx_t + derivs.ez_y
    res3 = derivs.hy_t - derivs.ez_x
    return res1, res2, res3


def energy_residual(fields: FieldBatch, derivs: FieldDerivs, eps):
    ez, hx, hy = fields.ez, fields.hx, fields.hy
    rate = eps * ez * derivs.ez_t + hx * derivs.hx_t + hy * derivs.hy_t
    flux_x = derivs.ez_x * hy + ez * derivs.hy_x
    flux_y = derivs.ez_y * hx + ez * derivs.hx_y
    return rate - flux_x + flux_y


def time_bin_weights(bin_losses: Sequence[float], kappa: float = 1.0) -> np.ndarray:
    """Causal gating w_1 = 1, w_m = min(1, exp(-kappa sum_{j<m} L_j))."""
    losses = np.asarray(bin_losses, dtype=np.float64)
    w = np.ones(len(losses))
    cum = 0.0
    for m in range(1, len(losses)):
        cum += losses[m - 1]
        w[m] = min(1.0, np.exp(-kappa * cum))
    return w


def total_loss(phys, ic, sym, energy, energy_enabled: bool = True):
    out = phys + IC_WEIGHT * ic + SYM_WEIGHT * sym
    if energy_enabled:
        out = out + ENERGY_WEIGHT * energy
    return out


SYM_TERMS_VACUUM = (("ez", "x", 1.0), ("ez", "y", 1.0), ("hx", "x", 1.0), ("hx", "y", -1.0),
                    ("hy", "x", -1.0), ("hy", "y", 1.0))
SYM_TERMS_DIELECTRIC = (("ez", "y", 1.0), ("hx", "y", -1.0), ("hy", "y", 1.0))


def sym_terms_for_case(case: str):
    if case == "vacuum":
        return SYM_TERMS_VACUUM
    if case == "dielectric":
        return SYM_TERMS_DIELECTRIC
    return ()


@dataclass
class LossBreakdown:
    phys: float
    ic: float
    sym: float
    energy: float
    total: float
    bin_phys: tuple = (0.0,) * M_BINS


@dataclass
class EpochEval:
    breakdown: LossBreakdown
    grad: Optional[torch.Tensor] = None


@dataclass
class _DevChunk:
    slices: list
    x: torch.Tensor
    y: torch.Tensor
    t: torch.Tensor
    bins: torch.Tensor
    is_ic: torch.Tensor
    spec: N.LossSpec = field(default=None)
    xyt: torch.Tensor = field(default=None)  # [3, R]; x, y, t are its rows (one H2D copy)


class _LossFn(torch.autograd.Function):
    """K4 forward computes the loss gradient too; backward just scales it."""

    @staticmethod
    def forward(ctx, out, dout, ev, chunk, weights_dev, sums, bd):
        R = out.shape[0]
        g_out = torch.empty_like(out)
        g_dout = torch.empty_like(dout)
        lib = N.lib()
        st = N.stream_ptr()
        with N.timed("loss"):
            N.check(lib.qpinn_loss_forward_backward(
                C.byref(chunk.spec), N.dtype_code(out.dtype), R, N.ptr(out), N.ptr(dout),
                N.ptr(weights_dev), N.ptr(g_out), N.ptr(g_dout), N.ptr(sums),
                N.ptr(ev._ws), ev._ws.numel(), st), "qpinn_loss_forward_backward")
        # this chunk's contribution to the total loss (finalize on the chunk sums)
        N.check(lib.qpinn_loss_finalize(C.byref(chunk.spec), N.ptr(sums), N.ptr(weights_dev),
                                        int(weights_dev is not None), 1.0, N.ptr(bd), None, st),
                "qpinn_loss_finalize")
        N.count_launches(3)
        ctx.save_for_backward(g_out, g_dout)
        return bd[4].clone()

    @staticmethod
    def backward(ctx, g):
        g_out, g_dout = ctx.saved_tensors
        g = g.to(g_out.dtype)
        return g_out * g, g_dout * g, None, None, None, None, None


class LossEvaluator:
    """All loss terms over a collocation grid in one fused device sweep.

    Same constructor surface as physics.py:274-315.  ``slices`` restricts the
    evaluator to a shard of whole time slices (data parallelism);
    ``max_points`` bounds one kernel sweep (chunks are whole slices, never
    straddling a time bin, exactly like the reference's chunks).
    """

    def __init__(self, model: Model, grid: CollocationGrid, material: MaterialMap, *,
                 case: Optional[str] = None, phys_mode: Optional[str] = None,
                 energy_enabled: bool = True, pulse: Optional[PulseSpec] = None,
                 chunk_slices: int = 4, bin_chunks: bool = True,
                 slices: Optional[Sequence[int]] = None, max_points: int = 1 << 21):
        self.model = model
        self.grid = grid
        self.material = material
        self.case = case or material.case
        if phys_mode is None:
            phys_mode = "diel_balanced" if self.case == "dielectric" else "vac"
        if phys_mode not in PHYS_MODES:
            raise ConfigError(f"unknown physics loss mode {phys_mode!r}")
        self.phys_mode = phys_mode
        self.energy_enabled = energy_enabled
        self.pulse = pulse or PulseSpec.for_case(self.case)
        self.sym_terms = sym_terms_for_case(self.case)
        self.chunk_slices = chunk_slices
        self.bin_chunks = bin_chunks
        s = grid.slice_size
        self.eps_slice = material.epsilon_at(grid.x_slice, grid.y_slice)
        self.vac_local = np.flatnonzero(self.eps_slice == 1.0)
        self.diel_local = np.flatnonzero(self.eps_slice != 1.0)
        if self.phys_mode == "diel_balanced" and self.diel_local.size == 0:
            raise ConfigError("diel_balanced mode requires dielectric points")
        self.ic_target = self.pulse.ez0(grid.x_slice, grid.y_slice)
        self.bin_slices = np.array([grid.bin_of_slice(i) for i in range(grid.nt)])
        self.bin_counts = np.array([(self.bin_slices == m).sum() * s for m in range(M_BINS)],
                                   dtype=np.int64)
        self.balanced = self.phys_mode == "diel_balanced"
        self.keys = KEYS_BAL if self.balanced else KEYS_VAC
        dev, dt = model.device, model.dtype
        self.device, self.dtype = dev, dt
        self._eps_dev = torch.as_tensor(self.eps_slice, dtype=torch.float64, device=dev)
        self._ic_dev = torch.as_tensor(self.ic_target, dtype=torch.float64, device=dev)
        # static normalisers (physics.py:432-450)
        inv_bin = np.zeros((M_BINS, 4))
        inv_all = np.zeros(4)
        for key in self.keys:
            k = _KEY_SLOT[key]
            for m in range(M_BINS):
                n_sl = int((self.bin_slices == m).sum())
                c = self._region_count(key, n_sl)
                inv_bin[m, k] = 1.0 / c if c else 0.0
            inv_all[k] = 1.0 / self._region_count(key, grid.nt)
        self._inv_bin, self._inv_all = inv_bin, inv_all
        keep = list(range(grid.nt)) if slices is None else sorted(int(v) for v in slices)
        self.slices = keep
        self.n_local_points = len(keep) * s
        self.chunks = self._make_chunks(keep, max(1, max_points // s))
        self._ws = torch.empty(N.lib().qpinn_loss_workspace_bytes(None, 0, 0), dtype=torch.uint8,
                               device=dev)
        self._sums_chunk = torch.zeros(N.LOSS_NSUMS, dtype=torch.float64, device=dev)
        self._bd_chunk = torch.zeros(10, dtype=torch.float64, device=dev)

    def _region_count(self, key: str, n_slices: int) -> int:
        s = self.grid.slice_size
        if key == "res1_vac":
            return n_slices * self.vac_local.size
        if key == "res1_diel":
            return n_slices * self.diel_local.size
        return n_slices * s

    def _make_chunks(self, keep, max_slices):
        """Whole-slice chunks that never straddle a time bin (physics.py:305-315)."""
        groups = []
        if self.bin_chunks:
            for m in range(M_BINS):
                sl = [v for v in keep if self.bin_slices[v] == m]
                if sl:
                    groups.append(sl)
        else:
            groups = [keep] if keep else []
        # merge bins into as few sweeps as max_slices allows (order preserved)
        merged, cur = [], []
        for g in groups:
            for lo in range(0, len(g), max_slices):
                part = g[lo:lo + max_slices]
                if len(cur) + len(part) > max_slices and cur:
                    merged.append(cur)
                    cur = []
                cur = cur + part
        if cur:
            merged.append(cur)
        return [self._dev_chunk(c) for c in merged]

    def _dev_chunk(self, sl):
        g, dev, dt = self.grid, self.device, self.dtype
        k = len(sl)
        xyt = torch.as_tensor(np.stack([np.tile(g.x_slice, k), np.tile(g.y_slice, k),
                                        np.repeat(g.ts[sl], g.slice_size)]), dtype=dt, device=dev)
        bins = torch.as_tensor(self.bin_slices[sl].astype(np.int32), device=dev)
        is_ic = torch.as_tensor((np.asarray(sl) == 0).astype(np.int32), device=dev)
        ch = _DevChunk(list(sl), xyt[0], xyt[1], xyt[2], bins, is_ic, xyt=xyt)
        ch.spec = self._spec(ch)
        return ch

    def _spec(self, ch: _DevChunk) -> N.LossSpec:
        sp = N.LossSpec()
        sp.nx, sp.ny, sp.n_local_slices = self.grid.nx, self.grid.ny, len(ch.slices)
        sp.slice_bin, sp.slice_is_ic = ch.bins.data_ptr(), ch.is_ic.data_ptr()
        sp.eps, sp.ic_target = self._eps_dev.data_ptr(), self._ic_dev.data_ptr()
        sp.balanced = int(self.balanced)
        sp.energy = int(self.energy_enabled)
        sp.n_sym = len(self.sym_terms)
        for i, (name, axis, sign) in enumerate(self.sym_terms):
            sp.sym_field[i] = {"ez": 0, "hx": 1, "hy": 2}[name]
            sp.sym_axis[i] = 0 if axis == "x" else 1
            sp.sym_sign[i] = sign
        for m in range(M_BINS):
            for k in range(4):
                sp.inv_count_bin[m][k] = self._inv_bin[m, k]
        for k in range(4):
            sp.inv_count_all[k] = self._inv_all[k]
        sp.n_total = float(self.grid.n_points)
        sp.slice_size = float(self.grid.slice_size)
        return sp

    def _weights_dev(self, weights):
        if weights is None:
            return None
        if torch.is_tensor(weights):
            return weights.to(device=self.device, dtype=torch.float64)
        return torch.as_tensor(np.asarray(weights, dtype=np.float64), device=self.device)

    @property
    def engine(self):
        """Native trunk/K1/K4/K2 sweep (hybrid models); None for classical variants."""
        if not hasattr(self, "_engine"):
            from .engine import NativeEngine
            self._engine = NativeEngine(self.model, self) if self.model.circuit is not None \
                else None
        return self._engine

    def sweep_native(self, flat: torch.Tensor, grad: Optional[torch.Tensor], weights_dev,
                     tape: bool, sums_out: torch.Tensor) -> None:
        """All-native sweep: gradient into ``grad`` (when tape), sums into ``sums_out``."""
        if weights_dev is not None and not self.bin_chunks:
            raise ConfigError("time-bin weights require bin_chunks=True")
        self.engine.sweep(flat, grad, weights_dev, sums_out, tape)

    def sweep(self, flat: torch.Tensor, weights_dev: Optional[torch.Tensor], tape: bool,
              sums_out: torch.Tensor) -> None:
        """Autograd sweep (torch trunk + K1/K2/K4 autograd functions): backward into
        ``flat.grad`` when tape; raw loss sums accumulate into ``sums_out``.  Used
        for classical variants and as an independent cross-check of the native
        engine."""
        if weights_dev is not None and not self.bin_chunks:
            raise ConfigError("time-bin weights require bin_chunks=True")
        for ch in self.chunks:
            with torch.set_grad_enabled(tape):
                out, dout = self.model.forward_raw(flat, ch.x, ch.y, ch.t)
                loss = _LossFn.apply(out, dout, self, ch, weights_dev, self._sums_chunk,
                                     self._bd_chunk)
            if tape:
                loss.backward()
            sums_out += self._sums_chunk

    def finalize(self, sums: torch.Tensor, weights_dev, kappa: float = 1.0,
                 bd_out: Optional[torch.Tensor] = None, weights_next: Optional[torch.Tensor] = None):
        bd = bd_out if bd_out is not None else torch.empty(10, dtype=torch.float64, device=self.device)
        spec = self.chunks[0].spec if self.chunks else self._spec(
            _DevChunk([], *(torch.empty(0, device=self.device),) * 3,
                      torch.zeros(1, dtype=torch.int32, device=self.device),
                      torch.zeros(1, dtype=torch.int32, device=self.device)))
        N.check(N.lib().qpinn_loss_finalize(C.byref(spec), N.ptr(sums), N.ptr(weights_dev),
                                            int(weights_dev is not None), kappa, N.ptr(bd),
                                            N.ptr(weights_next), N.stream_ptr()),
                "qpinn_loss_finalize")
        N.count_launches(1)
        return bd

    @staticmethod
    def breakdown_from(bd_host) -> LossBreakdown:
        v = [float(x) for x in bd_host]
        return LossBreakdown(phys=v[0], ic=v[1], sym=v[2], energy=v[3], total=v[4],
                             bin_phys=tuple(v[5:10]))

    def initial_bin_losses(self, params: ParameterStore) -> np.ndarray:
        return np.asarray(self.evaluate(params).breakdown.bin_phys)

    def evaluate(self, params, weights=None, tape: bool = False,
                 reduce_fn: Optional[Callable[[torch.Tensor], None]] = None,
                 native: bool = True) -> EpochEval:
        """One full pass (physics.py:334-428); grad is a device tensor when tape.
        ``native=False`` runs the autograd cross-check path instead."""
        flat_src = params.flat if isinstance(params, ParameterStore) else params
        wd = self._weights_dev(weights)
        sums = torch.zeros(N.LOSS_NSUMS, dtype=torch.float64, device=self.device)
        if native and self.engine is not None:
            flat = flat_src.detach().contiguous()
            grad = torch.empty_like(flat) if tape else None
            self.sweep_native(flat, grad, wd, tape, sums)
        else:
            flat = flat_src.detach().clone().requires_grad_(tape)
            self.sweep(flat, wd, tape, sums)
            grad = flat.grad if tape else None
            if tape and grad is None:
                grad = torch.zeros_like(flat)
        if reduce_fn is not None:
            packed = torch.cat([grad.double() if tape else sums.new_zeros(0), sums])
            reduce_fn(packed)
            if tape:
                grad = packed[:grad.numel()].to(grad.dtype)
            sums = packed[-N.LOSS_NSUMS:]
        bd = self.finalize(sums, wd)
        if self.model.circuit is not None:
            from .ansatz import check_domain
            check_domain(self.model.circuit, self.dtype, self.device,
                         ws=self.engine.pqc_ws if native and self.engine is not None else None)
        return EpochEval(self.breakdown_from(bd.cpu().numpy()), grad)
