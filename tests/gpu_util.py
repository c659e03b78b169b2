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
