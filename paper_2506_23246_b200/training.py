"""Training orchestration on the device: one fused step per epoch.

Mirrors ``qpinn.training`` (training.py): ``TrainConfig`` (:30-66),
``init_quantum_params`` (:69-79), ``lr_at`` (:82-84), ``AdamState`` /
``adam_step`` (:87-111), ``RunLog`` (:220-265) and ``train`` (:309-414).

The epoch step is device-resident: K1/K4/K2 plus the torch trunk produce the
gradient into the flat parameter tensor, the loss breakdown and the next
adaptive weights are finalised on the device, Adam runs in place with its
non-finite guard, and the host reads one small pinned record per step.
With ``world_size > 1`` every rank owns a contiguous block of whole time
slices; the packed [gradient | 23 loss sums] vector is all-reduced once
(NCCL over NVLink) before finalisation, which is exact.
Probes (Meyer-Wallach, energy history, L2 vs FDTD) are diagnostics off the
step path and are not part of this engine.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field, replace
from typing import Callable, List, Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, DomainError, RunAborted
from .network import Model, ModelConfig, ParameterStore, build_model, save_checkpoint
from .physics import (CollocationGrid, LossBreakdown, LossEvaluator, MaterialMap, default_t_end,
                      time_bin_weights)

INIT_STRATEGIES = ("reg", "zeros", "pi", "pi_half")


@dataclass
class TrainConfig:
    case: str = "vacuum"
    model: ModelConfig = field(default_factory=lambda: ModelConfig(
        variant="hybrid", ansatz="strongly", scale="acos"))
    energy_loss_enabled: bool = True
    phys_loss_mode: Optional[str] = None
    epochs: int = 1000
    lr0: float = 1e-3
    lr_decay: float = 0.85
    lr_decay_every: int = 2000
    seed: int = 0
    init_strategy: str = "reg"
    grid: tuple = (64, 64, 64)
    t_end: Optional[float] = None
    eps_r: float = 4.0
    slab_x0: float = 0.3
    eval_cadence: int = 250
    probe_cadence: int = 25
    probe_grid: tuple = (64, 64, 32)
    mw_probe_points: int = 32
    adaptive_weighting: bool = True
    kappa: float = 1.0
    chunk_slices: int = 4

    def __post_init__(self):
        if self.lr0 <= 0:
            raise ConfigError("lr0 must be positive")
        if self.epochs < 1:
            raise ConfigError("epochs must be >= 1")
        if self.init_strategy not in INIT_STRATEGIES:
            raise ConfigError(f"unknown init strategy {self.init_strategy!r}")
        if self.case not in ("vacuum", "dielectric", "asymmetric"):
            raise ConfigError(f"unknown case {self.case!r}")

    def resolved_t_end(self) -> float:
        return self.t_end if self.t_end is not None else default_t_end(self.case)


def init_quantum_params(strategy: str, count: int, seed: int = 0) -> np.ndarray:
    """training.py:69-79 (same numpy stream, float64)."""
    if strategy == "reg":
        return np.random.default_rng(seed).uniform(0.0, 2.0 * np.pi, count)
    if strategy == "zeros":
        return np.zeros(count)
    if strategy == "pi":
        return np.full(count, np.pi)
    if strategy == "pi_half":
        return np.full(count, np.pi / 2.0)
    raise ConfigError(f"unknown init strategy {strategy!r}")


def lr_at(epoch: int, lr0: float = 1e-3, decay: float = 0.85, every: int = 2000) -> float:
    return lr0 * decay ** (epoch // every)


@dataclass
class AdamState:
    """Device-resident Adam moments (training.py:87-98)."""
    m: torch.Tensor
    v: torch.Tensor
    t: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    @classmethod
    def zeros_like(cls, flat: torch.Tensor) -> "AdamState":
        return cls(m=torch.zeros_like(flat), v=torch.zeros_like(flat))


def adam_step(params: ParameterStore, grad: torch.Tensor, state: AdamState, lr: float,
              loss_dev: Optional[torch.Tensor] = None, flag: Optional[torch.Tensor] = None,
              sync: bool = True, veto: Optional[torch.Tensor] = None) -> None:
    """Bias-corrected Adam in place (training.py:101-111); RunAborted on a
    non-finite gradient (or loss) with params and state untouched.  A non-zero
    device ``veto`` (the step's reduced domain flag) skips the update the same
    way and raises DomainError, as the reference's forward does before any
    update (ansatz.py:51-58)."""
    flat = params.flat if isinstance(params, ParameterStore) else params
    if flag is None:
        flag = torch.zeros(1, dtype=torch.int32, device=flat.device)
    N.check(N.lib().qpinn_adam_step(
        N.dtype_code(flat.dtype), flat.numel(), N.ptr(flat), N.ptr(grad.contiguous()),
        N.ptr(state.m), N.ptr(state.v), state.t + 1, lr, state.beta1, state.beta2, state.eps,
        N.ptr(loss_dev), N.ptr(veto), N.ptr(flag), N.stream_ptr()), "qpinn_adam_step")
    N.count_launches(2)
    if sync:
        f = int(flag.item())
        if f & 4:
            raise DomainError("scale input exceeds [-1, 1] by more than 1e-12")
        if f:
            raise RunAborted("non-finite gradient" if f & 1 else "non-finite loss")
        state.t += 1


# -- data parallelism over whole time slices ------------------------------------

def shard_slices(nt: int, rank: int, world: int) -> List[int]:
    """Contiguous, balanced block of whole time slices for ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError("bad rank/world")
    base, extra = divmod(nt, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return list(range(lo, hi))


def allreduce_fn(group=None) -> Callable[[torch.Tensor], None]:
    """In-place sum all-reduce of the packed [grad | sums] vector."""
    import torch.distributed as dist

    def fn(t: torch.Tensor) -> None:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return fn


def reduce_packed(grad: Optional[torch.Tensor], sums: torch.Tensor, reduce_fn,
                  packed: Optional[torch.Tensor] = None, extra: Optional[torch.Tensor] = None):
    """Pack (grad as float64, sums, extra), reduce once, unpack in place.
    ``extra`` carries the step's domain flags (``qpinn_pqc_domain_flags``), so
    a DomainError on any rank is seen -- and raised -- by every rank."""
    parts = [t for t in (grad, sums, extra) if t is not None]
    sizes = [t.numel() for t in parts]
    if packed is None or packed.numel() != sum(sizes):
        packed = torch.empty(sum(sizes), dtype=torch.float64, device=sums.device)
    o = 0
    for t, k in zip(parts, sizes):
        packed[o:o + k].copy_(t.reshape(-1))
        o += k
    reduce_fn(packed)
    o = 0
    for t, k in zip(parts, sizes):
        t.reshape(-1).copy_(packed[o:o + k])
        o += k
    return packed


def raise_domain(err: float, clamped: float, max_abs: float) -> None:
    """The reference domain rule (ansatz.py:51-58) on the step's (reduced) flags."""
    if err > 0.0:
        raise DomainError(f"scale input exceeds [-1, 1] by more than 1e-12 on "
                          f"{int(round(err))} rank(s) (max |a| here {max_abs:.17g})")
    if clamped > 0.0:
        import warnings
        warnings.warn("scale input clamped into [-1, 1] (excursion <= 1e-12)", stacklevel=3)


# -- run log -------------------------------------------------------------------------

CSV_COLUMNS = ("epoch", "lr", "phys", "ic", "sym", "energy", "total",
               "grad_norm_all", "grad_var_all", "grad_norm_q", "grad_var_q",
               "mw_q", "i_bh", "l2_err")


@dataclass
class RunRow:
    epoch: int
    lr: float
    phys: float
    ic: float
    sym: float
    energy: float
    total: float
    grad_norm_all: Optional[float] = None
    grad_var_all: Optional[float] = None
    grad_norm_q: Optional[float] = None
    grad_var_q: Optional[float] = None
    mw_q: Optional[float] = None
    i_bh: Optional[float] = None
    l2_err: Optional[float] = None
    bin_phys: tuple = ()

    def csv_cells(self):
        def fmt(v):
            return "" if v is None else repr(v)
        return [str(self.epoch)] + [fmt(v) for v in
                (self.lr, self.phys, self.ic, self.sym, self.energy, self.total,
                 self.grad_norm_all, self.grad_var_all, self.grad_norm_q,
                 self.grad_var_q, self.mw_q, self.i_bh, self.l2_err)]


@dataclass
class RunLog:
    """training.py:236-252."""
    rows: List[RunRow] = field(default_factory=list)
    wall_s: float = 0.0
    final_i_bh: Optional[float] = None
    final_i_bh_raw: Optional[float] = None
    final_l2: Optional[float] = None
    energy_history: Optional[np.ndarray] = None

    def to_csv(self, path) -> None:
        with open(path, "w") as f:
            f.write(",".join(CSV_COLUMNS) + "\n")
            for row in self.rows:
                f.write(",".join(row.csv_cells()) + "\n")


@dataclass
class TrainResult:
    log: RunLog
    model: Model
    params: ParameterStore

    def summary(self, config: "TrainConfig", thresholds=None) -> dict:
        """training.py:264-300."""
        from .probes import detect_collapse
        last = self.log.rows[-1]
        report = detect_collapse(self.log, thresholds) if self.log.final_i_bh is not None \
            else None
        return {
            "case": config.case, "variant": config.model.variant,
            "ansatz": config.model.ansatz, "scale": config.model.scale,
            "energy_loss_enabled": config.energy_loss_enabled, "seed": config.seed,
            "epochs": len(self.log.rows),
            "counts": {"classical": self.model.n_classical, "quantum": self.model.n_quantum,
                       "total": self.model.total_parameter_count},
            "final": {"phys": last.phys, "ic": last.ic, "sym": last.sym,
                      "energy": last.energy, "total": last.total},
            "first_total": self.log.rows[0].total,
            "final_l2": self.log.final_l2, "i_bh": self.log.final_i_bh,
            "i_bh_raw": self.log.final_i_bh_raw,
            "collapsed": report.collapsed if report else None,
            "wall_s": self.log.wall_s,
        }


# -- the step engine ---------------------------------------------------------------------

def _graph_kernel_nodes(g) -> Optional[int]:
    """Kernel nodes of a captured step graph (cuda-python on the raw cudaGraph_t; the
    step's own kernels plus the few torch elementwise ops inside it); None when the
    bindings are unavailable."""
    try:
        import cuda.bindings.runtime as rt
        graph = rt.cudaGraph_t(init_value=int(g.raw_cuda_graph()))
        err, _, n = rt.cudaGraphGetNodes(graph, 0)
        if err != rt.cudaError_t.cudaSuccess:
            return None
        err, nodes, n = rt.cudaGraphGetNodes(graph, n)
        if err != rt.cudaError_t.cudaSuccess:
            return None
        k = 0
        for nd in nodes[:n]:
            err, t = rt.cudaGraphNodeGetType(nd)
            if err == rt.cudaError_t.cudaSuccess and t == rt.cudaGraphNodeType.cudaGraphNodeTypeKernel:
                k += 1
        return k
    except Exception:  # noqa: BLE001 - instrumentation only
        return None


class Trainer:
    """Device-resident QPINN epoch step (training.py:359-407; probes run in ``train``)."""

    def __init__(self, config: TrainConfig, device="cuda", dtype=torch.float32,
                 rank: int = 0, world_size: int = 1, reduce_fn=None, log_grad: bool = False,
                 max_points: int = 1 << 21, graphs: bool = True):
        self.config = config
        self.device = torch.device(device)
        t_end = config.resolved_t_end()
        self.model = build_model(replace(config.model, t_domain=t_end), device=device, dtype=dtype)
        flat = self.model.init_params_np()
        if self.model.n_quantum:
            flat[self.model.n_classical:] = init_quantum_params(
                config.init_strategy, self.model.n_quantum, config.seed)
        self.params = self.model.params_from(flat)
        self.flat = self.params.flat
        self.grad = torch.zeros_like(self.flat)
        nx, ny, nt = config.grid
        self.grid = CollocationGrid(nx, ny, nt, t_end)
        self.material = MaterialMap(case=config.case, eps_r=config.eps_r, slab_x0=config.slab_x0)
        self.world_size, self.rank = world_size, rank
        self.slices = shard_slices(nt, rank, world_size)
        self.reduce_fn = reduce_fn if world_size > 1 else None
        self.evaluator = LossEvaluator(
            self.model, self.grid, self.material, case=config.case,
            phys_mode=config.phys_loss_mode, energy_enabled=config.energy_loss_enabled,
            chunk_slices=config.chunk_slices, slices=self.slices, max_points=max_points)
        self.adam = AdamState.zeros_like(self.flat.detach())
        dev = self.device
        self.sums = torch.zeros(N.LOSS_NSUMS, dtype=torch.float64, device=dev)
        self.bd = torch.zeros(10, dtype=torch.float64, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        # [DomainError flag, clamp flag, max|a|] of the step's forwards (device)
        self.dom = torch.zeros(3, dtype=torch.float64, device=dev)
        self.weights = None
        self.weights_next = None
        self._packed = None
        self.log_grad = log_grad
        self._host = torch.zeros(20, dtype=torch.float64, pin_memory=True)
        self._host_flag = torch.zeros(1, dtype=torch.int32, pin_memory=True)  # same dtype: a plain D2H
        if config.adaptive_weighting:
            # untaped initial pass (training.py:336-339)
            bins = self._evaluate_untaped()
            self.weights = torch.as_tensor(time_bin_weights(bins, config.kappa),
                                           dtype=torch.float64, device=dev)
            self.weights_next = torch.empty_like(self.weights)
        self.epoch = 0
        self._host_inputs = None
        # CUDA graphs of the step's local sweep (native engine): one graph per
        # (bin-weight buffer, input mode); captured after a warm step
        self.use_graphs = graphs and dev.type == "cuda" and self.evaluator.engine is not None
        self._graphs = {}

    # -- end-to-end mode: collocation inputs come from pinned host memory ------
    def set_host_inputs(self, on: bool) -> None:
        """End-to-end mode: every step's collocation inputs come from pinned host
        memory, one [3, R] H2D copy per chunk.  The device inputs are double
        buffered: step k runs on buffer k % 2 while the copy of step k+1's inputs
        fills the other buffer on a side stream (an input pipeline's prefetch;
        each step still moves its own inputs host -> device)."""
        if self._host_inputs is not None:
            self._bind_inputs(0)
        if not on:
            self._host_inputs = None
            return
        chunks = self.evaluator.chunks
        self._host_inputs = [ch.xyt.detach().cpu().pin_memory() for ch in chunks]
        self._in_bufs = [(ch.xyt, torch.empty_like(ch.xyt)) for ch in chunks]
        self._in_par = 0
        self._copy_stream = torch.cuda.Stream(device=self.device)
        self._copy_done = [torch.cuda.Event(), torch.cuda.Event()]
        for (b0, _), h in zip(self._in_bufs, self._host_inputs):  # the first step's inputs
            b0.copy_(h)
        torch.cuda.current_stream().synchronize()
        self._copy_pending = [False, False]

    def _bind_inputs(self, par: int) -> None:
        for ch, bufs in zip(self.evaluator.chunks, self._in_bufs):
            b = bufs[par]
            ch.xyt, ch.x, ch.y, ch.t = b, b[0], b[1], b[2]

    def _use_inputs(self) -> int:
        """Bind this step's input buffer (waiting for its copy); returns its parity."""
        par = self._in_par
        if self._copy_pending[par]:
            torch.cuda.current_stream().wait_event(self._copy_done[par])
            self._copy_pending[par] = False
        self._bind_inputs(par)
        return par

    def _prefetch_inputs(self) -> None:
        """Start the next step's H2D copy into the other buffer (enqueued after this
        step's launches, so the host work overlaps the device work); the other
        buffer's last reader, the previous step, has finished: step() synchronises."""
        nxt = 1 - self._in_par
        with torch.cuda.stream(self._copy_stream):
            for bufs, h in zip(self._in_bufs, self._host_inputs):
                bufs[nxt].copy_(h, non_blocking=True)
            self._copy_done[nxt].record(self._copy_stream)
        self._copy_pending[nxt] = True
        self._in_par = nxt

    def host_input_bytes(self) -> int:
        if not self._host_inputs:
            return 0
        return sum(v.numel() * v.element_size() for v in self._host_inputs)

    def readback_bytes(self) -> int:
        return 10 * 8 + 4 + 3 * 8 + (32 if self.log_grad else 0)  # loss record, flag, domain

    def _evaluate_untaped(self):
        sums = torch.zeros(N.LOSS_NSUMS, dtype=torch.float64, device=self.device)
        self._sweep(None, None, False, sums)
        self._domain_flags()
        if self.reduce_fn is not None:
            reduce_packed(None, sums, self.reduce_fn, extra=self.dom[:2])
        bd = self.evaluator.finalize(sums, None)
        d = self.dom.cpu().numpy()
        raise_domain(d[0], d[1], d[2])
        return bd[5:10].cpu().numpy()

    def _sweep(self, grad, weights, tape, sums):
        if self.evaluator.engine is not None:
            self.evaluator.sweep_native(self.flat, grad, weights, tape, sums)
            return grad
        flat = self.flat.detach().requires_grad_(tape)
        with torch.set_grad_enabled(tape):
            self.evaluator.sweep(flat, weights, tape, sums)
        if tape:
            grad.copy_(flat.grad)
        return grad

    def _local_sweep(self):
        """The sweep (forward + backward) over this rank's chunks."""
        eng = self.evaluator.engine
        if eng is None or len(eng.chunks) > 1:  # one native chunk overwrites the sums
            self.sums.zero_()
        return self._sweep(self.grad, self.weights, True, self.sums)

    def _pqc_workspace(self):
        """The workspace whose running max|a| this trainer's forwards fold into."""
        eng = self.evaluator.engine
        if eng is not None:
            return eng.pqc_ws
        return self.model.circuit.workspace(self.model.dtype, self.device, 0)

    def _domain_flags(self):
        """[error, clamp, max|a|] of the forwards since the last call, on the device."""
        if self.model.circuit is None:
            return
        N.check(N.lib().qpinn_pqc_domain_flags(C.c_void_p(self._pqc_workspace().data_ptr()),
                                               C.c_void_p(self.dom.data_ptr()),
                                               C.c_void_p(N.stream_ptr())), "domain flags")
        N.count_launches(1)

    def _reduce_finalize(self, grad):
        """The step's one collective (data parallel; it also carries the domain
        flags), then the loss finalisation."""
        self._domain_flags()
        if self.reduce_fn is not None:
            self._packed = reduce_packed(grad, self.sums, self.reduce_fn, self._packed,
                                         extra=self.dom[:2] if self.model.circuit is not None
                                         else None)
        self.evaluator.finalize(self.sums, self.weights, self.config.kappa, self.bd,
                                self.weights_next if self.weights is not None else None)

    def _device_part(self):
        """The device part of a step.  Once warm, the local sweep (the whole
        fixed launch sequence over preallocated buffers) replays from a CUDA
        graph; the collective and the finalisation run eagerly after it, so the
        NCCL all-reduce is never captured.  Eager throughout while per-kernel
        event timing is on."""
        par = self._use_inputs() if self._host_inputs is not None else -1
        if not self.use_graphs or self.epoch < 1 or N.timing_enabled():
            grad = self._local_sweep()
        else:
            key = (self.weights.data_ptr() if self.weights is not None else 0, par)
            entry = self._graphs.get(key)
            if entry is None:
                g = torch.cuda.CUDAGraph(keep_graph=True)
                l0 = N.LAUNCHES["count"]
                with torch.cuda.graph(g):
                    self._local_sweep()
                # launches per replay: the graph's kernel nodes when cuda-python can
                # read them, else the count the wrappers declared while capturing
                nodes = _graph_kernel_nodes(g)
                entry = (g, nodes if nodes is not None else N.LAUNCHES["count"] - l0)
                N.LAUNCHES["count"] = l0
                g.instantiate()
                self._graphs[key] = entry
            entry[0].replay()
            N.count_launches(entry[1])
            grad = self.grad
        if self._host_inputs is not None:
            self._prefetch_inputs()
        self._reduce_finalize(grad)
        return grad

    def step(self) -> RunRow:
        """One epoch: evaluate(tape=True) -> (all-reduce) -> finalize -> Adam."""
        cfg = self.config
        epoch = self.epoch
        lr = lr_at(epoch, cfg.lr0, cfg.lr_decay, cfg.lr_decay_every)
        grad = self._device_part()
        adam_step(self.flat, grad, self.adam, lr, loss_dev=self.bd[4:5], flag=self.flag,
                  sync=False, veto=self.dom[0:1] if self.model.circuit is not None else None)
        host = self._host
        host[:10].copy_(self.bd, non_blocking=True)
        self._host_flag.copy_(self.flag, non_blocking=True)
        if self.log_grad:
            g = grad.double()
            host[11] = 0.0
            host[11:12].copy_(torch.linalg.vector_norm(g).reshape(1), non_blocking=True)
            host[12:13].copy_(torch.var(g, unbiased=False).reshape(1), non_blocking=True)
            q = g[self.model.n_classical:]
            if q.numel():
                host[13:14].copy_(torch.linalg.vector_norm(q).reshape(1), non_blocking=True)
                host[14:15].copy_(torch.var(q, unbiased=False).reshape(1), non_blocking=True)
        host[15:18].copy_(self.dom, non_blocking=True)  # domain flags ride along
        torch.cuda.current_stream().synchronize()
        v = host.numpy()
        # the forward's DomainError comes first, as in the reference (Adam was vetoed)
        raise_domain(v[15], v[16], v[17])
        f = int(self._host_flag[0])
        if f:
            raise RunAborted(("non-finite loss" if f & 2 else "non-finite gradient")
                             + f" at epoch {epoch}; last good parameters preserved")
        self.adam.t += 1
        if self.weights is not None:
            self.weights, self.weights_next = self.weights_next, self.weights
        self.epoch += 1
        bd = LossEvaluator.breakdown_from(v[:10])
        row = RunRow(epoch=epoch, lr=lr, phys=bd.phys, ic=bd.ic, sym=bd.sym, energy=bd.energy,
                     total=bd.total, bin_phys=bd.bin_phys)
        if self.log_grad:
            row.grad_norm_all, row.grad_var_all = float(v[11]), float(v[12])
            if self.model.n_quantum:
                row.grad_norm_q, row.grad_var_q = float(v[13]), float(v[14])
        return row


def train(config: TrainConfig, reference=None, outdir=None, on_epoch=None, device="cuda",
          dtype=torch.float32, rank: int = 0, world_size: int = 1, reduce_fn=None) -> TrainResult:
    """Full-batch Adam training with the reference's probes (training.py:309-414).

    Per epoch, on the pre-update parameters as in the reference: the
    Meyer-Wallach Q on 32 seeded probe points (hybrid models), the energy
    probe and black-hole index every ``probe_cadence`` epochs and on the last,
    and the L2 error against ``reference`` (an FDTD ``FieldHistory``) every
    ``eval_cadence`` epochs and on the last.  Probes run on the native
    inference engine; on ranks > 0 of a data-parallel run they are skipped.
    """
    from .probes import bh_index, energy_probe, l2_against_reference, probe_entanglement
    if config.eval_cadence > 0 and reference is None:
        raise ConfigError("eval_cadence > 0 requires a reference solution "
                          "(set eval_cadence=0 to disable L2 evaluation)")
    t0 = time.perf_counter()
    tr = Trainer(config, device=device, dtype=dtype, rank=rank, world_size=world_size,
                 reduce_fn=reduce_fn, log_grad=True)
    t_end = config.resolved_t_end()
    prng = np.random.default_rng([config.seed, 9])  # training.py:342-345
    mw_x = prng.uniform(-1.0, 1.0, config.mw_probe_points)
    mw_y = prng.uniform(-1.0, 1.0, config.mw_probe_points)
    mw_t = prng.uniform(0.0, t_end, config.mw_probe_points)
    probe_times = np.linspace(0.0, t_end, config.probe_grid[2])
    probes_here = rank == 0
    log = RunLog()
    try:
        for epoch in range(config.epochs):
            last = epoch == config.epochs - 1
            mw = i_bh = l2 = None
            if probes_here and tr.model.n_quantum:
                mw = probe_entanglement(tr.model, tr.params, mw_x, mw_y, mw_t)
            if probes_here and config.probe_cadence > 0 and (
                    epoch % config.probe_cadence == 0 or last):
                u_hist = energy_probe(tr.model, tr.params, tr.material, config.probe_grid[0],
                                      config.probe_grid[1], probe_times)
                i_bh, raw = bh_index(u_hist, probe_times)
                log.final_i_bh, log.final_i_bh_raw = i_bh, raw
                log.energy_history = u_hist
            if probes_here and config.eval_cadence > 0 and reference is not None and (
                    epoch % config.eval_cadence == 0 or last):
                l2 = l2_against_reference(tr.model, tr.params, reference)
                log.final_l2 = l2
            row = tr.step()
            row.mw_q, row.i_bh, row.l2_err = mw, i_bh, l2
            log.rows.append(row)
            if on_epoch is not None:
                on_epoch(row)
    except RunAborted:
        log.wall_s = time.perf_counter() - t0
        if outdir is not None:
            import os
            save_checkpoint(os.path.join(str(outdir), "last_good.ckpt"), tr.model, tr.params)
            log.to_csv(os.path.join(str(outdir), "metrics.csv"))
        raise
    log.wall_s = time.perf_counter() - t0
    if outdir is not None:
        import os
        save_checkpoint(os.path.join(str(outdir), "final.ckpt"), tr.model, tr.params)
        log.to_csv(os.path.join(str(outdir), "metrics.csv"))
    return TrainResult(log=log, model=tr.model, params=tr.params)
