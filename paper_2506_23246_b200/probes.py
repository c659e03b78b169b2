"""Diagnostic probes on the native inference engine.

Mirrors the reference's probe API (training.py:117-217): the Meyer-Wallach
entanglement of the circuit state (qsim.py:384-406), the energy probe U(t)
on a collocated grid and its black-hole index, and the relative L2 error of
E_z against an FDTD field history.  The fields come from the value-only
engine (value trunk on the tensor cores, K1 without tangents, head kernel),
the per-slice energy and L2 sums from deterministic device reductions
(csrc/probes.cu); only the final few scalars are combined on the host.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .errors import MetricError


def _engine_inputs(model, params, x, y, t):
    x, y, t = model._coords(x, y, t)
    flat = params.flat if hasattr(params, "flat") else params
    return model.inference, flat.detach(), x.contiguous(), y.contiguous(), t.contiguous()


def probe_entanglement(model, params, x, y, t) -> Optional[float]:
    """Mean Meyer-Wallach Q of the circuit state at the probe inputs
    (training.py:174-184); None for classical variants."""
    if model.circuit is None:
        return None
    eng, flat, x, y, t = _engine_inputs(model, params, x, y, t)
    q = eng.meyer_wallach(flat, x, y, t)
    eng.check_domain()
    return float(q.mean().item())


def _grid_points(nx: int, ny: int):
    xs = -1.0 + 2.0 * np.arange(nx) / nx
    ys = -1.0 + 2.0 * np.arange(ny) / ny
    yy, xx = np.meshgrid(ys, xs, indexing="ij")
    return xx.ravel(), yy.ravel()


def _fields_on_slices(model, params, xf, yf, times):
    """Fields [T * P, 3] on the device for P = len(xf) points at each time."""
    T, P = len(times), len(xf)
    x = np.tile(xf, T)
    y = np.tile(yf, T)
    t = np.repeat(np.asarray(times, dtype=np.float64), P)
    eng, flat, xd, yd, td = _engine_inputs(model, params, x, y, t)
    out = eng.fields(flat, xd, yd, td)
    eng.check_domain()
    return out


def energy_probe(model, params, material, nx: int, ny: int, times) -> np.ndarray:
    """U_theta(t_k) on a collocated nx x ny grid decoupled from training
    (training.py:187-200)."""
    xf, yf = _grid_points(nx, ny)
    out = _fields_on_slices(model, params, xf, yf, times)
    eps = torch.as_tensor(material.epsilon_at(xf, yf), dtype=torch.float64, device=out.device)
    u = torch.empty(len(times), dtype=torch.float64, device=out.device)
    N.check(N.lib().qpinn_probe_energy(N.dtype_code(out.dtype), len(times), len(xf),
                                       out.data_ptr(), eps.data_ptr(), (2.0 / nx) * (2.0 / ny),
                                       u.data_ptr(), N.stream_ptr()), "qpinn_probe_energy")
    N.count_launches(1)
    return u.cpu().numpy()


def l2_against_reference(model, params, reference) -> float:
    """Relative L2 error of E_z on the reference snapshot grid (training.py:203-217)."""
    yy, xx = np.meshgrid(reference.ys, reference.xs, indexing="ij")
    xf, yf = xx.ravel(), yy.ravel()
    out = _fields_on_slices(model, params, xf, yf, reference.times)
    ref = torch.as_tensor(np.ascontiguousarray(reference.ez, dtype=np.float64).reshape(-1),
                          device=out.device)
    sums = torch.empty(2 * len(reference.times), dtype=torch.float64, device=out.device)
    N.check(N.lib().qpinn_probe_l2(N.dtype_code(out.dtype), len(reference.times), len(xf),
                                   out.data_ptr(), ref.data_ptr(), sums.data_ptr(),
                                   N.stream_ptr()), "qpinn_probe_l2")
    N.count_launches(1)
    s = sums.cpu().numpy()
    num = den = 0.0
    for k in range(len(reference.times)):  # the reference's accumulation order
        num += float(s[2 * k])
        den += float(s[2 * k + 1])
    if den == 0.0:
        raise MetricError("reference field has zero norm")
    return float(np.sqrt(num / den))


def bh_index(u_history: Sequence[float], times: Optional[Sequence[float]] = None):
    """(clamped, raw) black-hole index 1 - min_{t > 0} U(t)/U(0) (training.py:117-134)."""
    u = np.asarray(u_history, dtype=np.float64)
    if u[0] <= 0.0:
        raise MetricError("U(0) must be positive to normalize the energy history")
    u_tilde = u / u[0]
    mask = (np.asarray(times) > 0.0) if times is not None else (np.arange(len(u)) > 0)
    if not np.any(mask):
        raise MetricError("energy history needs at least one positive time")
    raw = 1.0 - float(np.min(u_tilde[mask]))
    return float(np.clip(raw, 0.0, 1.0)), raw


@dataclass
class CollapseThresholds:
    """I_BH >= i_bh with L_phys <= phys declares collapse (training.py:137-142)."""
    i_bh: float = 0.9
    phys: float = 1.0


@dataclass
class BHReport:
    i_bh: float
    collapsed: bool
    ensemble_bh: Optional[bool] = None


def detect_collapse(runlogs, thresholds: Optional[CollapseThresholds] = None) -> BHReport:
    """Collapse verdict for one RunLog or an ensemble (training.py:152-168)."""
    th = thresholds or CollapseThresholds()
    logs = runlogs if isinstance(runlogs, (list, tuple)) else [runlogs]
    flags, i_bhs = [], []
    for log in logs:
        i_bh = log.final_i_bh
        phys = log.rows[-1].phys
        if i_bh is None:
            raise MetricError("run has no energy probe; cannot assess collapse")
        flags.append(i_bh >= th.i_bh and phys <= th.phys)
        i_bhs.append(i_bh)
    if len(logs) == 1:
        return BHReport(i_bh=i_bhs[0], collapsed=flags[0], ensemble_bh=None)
    fraction = float(np.mean(flags))
    return BHReport(i_bh=float(np.max(i_bhs)), collapsed=all(flags),
                    ensemble_bh=fraction > 0.95)
