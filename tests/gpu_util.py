"""Shared helpers for the GPU parity tests."""
import numpy as np
import torch

# FP32 parity: |got - want| <= 1e-5 |want| + 1e-6 max|want| per output tensor
# (north_star 1e-5 relative; the absolute floor is the SURVEY 8.C finding that
# near-zero outputs cannot meet a pure relative bound in FP32).
F32_RTOL, F32_ATOL_FRAC = 1e-5, 1e-6
# FP64 verification build: 1e-10 relative (north_star)
F64_RTOL, F64_ATOL_FRAC = 1e-10, 1e-12


def tol(dtype):
    return (F64_RTOL, F64_ATOL_FRAC) if dtype == torch.float64 else (F32_RTOL, F32_ATOL_FRAC)


def assert_close(got, want, dtype, what="", scale=1.0):
    got = got.detach().double().cpu().numpy() if torch.is_tensor(got) else np.asarray(got)
    want = np.asarray(want, dtype=np.float64)
    rtol, af = tol(dtype)
    rtol, af = rtol * scale, af * scale
    atol = af * max(np.max(np.abs(want)), 1e-300)
    err = np.abs(got - want)
    bad = err > rtol * np.abs(want) + atol
    if bad.any():
        i = np.unravel_index(np.argmax(err / (rtol * np.abs(want) + atol)), err.shape)
        raise AssertionError(f"{what}: {bad.sum()} / {bad.size} entries out of tolerance; "
                             f"worst at {i}: got {got[i]!r} want {want[i]!r}")


def cuda(x, dtype):
    return torch.as_tensor(np.asarray(x), dtype=dtype, device="cuda").contiguous()


# FP32 error budget for ill-conditioned cases.  An FP32 implementation first
# rounds its inputs (activations, tangents, circuit parameters) to float32;
# evaluated EXACTLY (float64) on those rounded inputs, the outputs already
# differ from the float64 reference by the "input-rounding floor" -- which no
# FP32 kernel can beat.  Near |a| -> 1 the acos/asin embedding amplifies it by
# S'(a) = 1/sqrt(1 - a^2) and S''(a) = a/(1 - a^2)^1.5, so a fixed
# 1e-6 * max floor is meaningless there.  The budget per output tensor is
#   |got - want| <= 1e-5 |want| + max(1e-6 max|want|, FLOOR_FACTOR * floor)
# with floor = max |f64(round32(inputs)) - f64(inputs)| computed by the oracle
# on the same inputs, and FLOOR_FACTOR the allowance for the kernels' own
# FP32 arithmetic (measured 1.5-3x the floor on the bench chain,
# scripts/fp32_error_budget.py -> profiles/r02/fp32_error_budget.json).
FLOOR_FACTOR = 4.0


def round32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def input_rounding_floor(fn, *inputs):
    """Per-output max |fn(round32(inputs)) - fn(inputs)| (fn: oracle, float64)."""
    exact = fn(*inputs)
    rounded = fn(*(round32(x) for x in inputs))
    return [float(np.max(np.abs(np.asarray(r) - np.asarray(e)))) if np.size(e) else 0.0
            for r, e in zip(rounded, exact)]


def assert_close_budget(got, want, dtype, floor, what=""):
    """assert_close with the FP32 input-rounding-floor budget (float64: 1e-10)."""
    if dtype == torch.float64:
        return assert_close(got, want, dtype, what)
    got = got.detach().double().cpu().numpy() if torch.is_tensor(got) else np.asarray(got)
    want = np.asarray(want, dtype=np.float64)
    atol = max(F32_ATOL_FRAC * max(np.max(np.abs(want)), 1e-300), FLOOR_FACTOR * floor)
    err = np.abs(got - want)
    bad = err > F32_RTOL * np.abs(want) + atol
    if bad.any():
        i = np.unravel_index(np.argmax(err / (F32_RTOL * np.abs(want) + atol)), err.shape)
        raise AssertionError(f"{what}: {bad.sum()} / {bad.size} entries outside the FP32 budget "
                             f"(floor {floor:.3e}); worst at {i}: got {got[i]!r} want {want[i]!r}")


def norm_rel(got, want):
    got = got.detach().double().cpu().numpy() if torch.is_tensor(got) else np.asarray(got)
    want = np.asarray(want, dtype=np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))
