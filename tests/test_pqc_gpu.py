"""K1/K2 parity on the GPU through the C ABI, against reference golden vectors
and the numpy oracle."""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import golden_cases
from gpu_util import assert_close, assert_close_budget, cuda, input_rounding_floor

pytestmark = pytest.mark.gpu
DTYPES = [torch.float64, torch.float32]


def _run(d, kind, scale, L, dtype):
    from paper_2506_23246_b200.ansatz import build_circuit, pqc_backward_raw, pqc_forward_raw
    n = d["a"].shape[1]
    c = build_circuit(kind, n, L)
    a, da, qp = cuda(d["a"], dtype), cuda(d["da"], dtype), cuda(d["qp"], dtype)
    z, dz = pqc_forward_raw(c, scale, a, da, qp)
    zp, _ = pqc_forward_raw(c, scale, a, None, qp)
    ga, gda, gq = pqc_backward_raw(c, scale, a, da, qp, cuda(d["gz"], dtype), cuda(d["gdz"], dtype))
    return z, dz, zp, ga, gda, gq


def _check_fixture(name, L_of, dtype):
    for key, d in golden_cases(name).items():
        parts = key.split("/")
        kind = parts[0]
        scale, L = L_of(parts)
        z, dz, zp, ga, gda, gq = _run(d, kind, scale, L, dtype)
        got = (z, dz, zp, ga, gda, gq)
        want = (d["z"], d["dz"], d["zplain"], d["ga"], d["gda"], d["gq"])
        names = ("z", "dz", "z(value-only)", "g_a", "g_da", "g_qparams")
        if "edge" in key:
            # |a| -> 0.995 amplifies input rounding by S'' ~ (1-a^2)^-1.5 ~ 1e3:
            # the FP32 budget is stated against the oracle's input-rounding floor
            fl = _floors(d, kind, scale, L)
            for x, w, nm, f in zip(got, want, names, fl):
                assert_close_budget(x, w, dtype, f, f"{key} {nm}")
        else:
            for x, w, nm in zip(got, want, names):
                assert_close(x, w, dtype, f"{key} {nm}")


def _floors(d, kind, scale, L):
    """Input-rounding floors (gpu_util) of z, dz, z, g_a, g_da, g_qparams."""
    fz = input_rounding_floor(lambda a, da, qp: O.pqc_forward(a, da, qp, kind, scale, L),
                              d["a"], d["da"], d["qp"])
    fb = input_rounding_floor(
        lambda a, da, qp, gz, gdz: O.pqc_backward(a, da, qp, kind, scale, L, gz, gdz),
        d["a"], d["da"], d["qp"], d["gz"], d["gdz"])
    return fz + [fz[0]] + fb


@pytest.mark.parametrize("dtype", DTYPES)
def test_pqc_all_ansatz_scale_small(dtype):
    _check_fixture("pqc_small.npz", lambda p: (p[1], 2), dtype)


@pytest.mark.parametrize("dtype", DTYPES)
def test_pqc_default_7q_4l(dtype):
    _check_fixture("pqc_n7.npz", lambda p: (p[1], 4), dtype)


@pytest.mark.parametrize("dtype", DTYPES)
def test_pqc_mid_sizes(dtype):
    _check_fixture("pqc_mid.npz", lambda p: ("bias", int(p[2])), dtype)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("n,L", [(1, 3), (2, 2), (8, 2)])
def test_pqc_vs_oracle_other_sizes(dtype, n, L):
    # float64 n = 8 is beyond the register kernels: it runs the global-memory path
    rng = np.random.default_rng(n * 100 + L)
    for kind in (("no_entanglement",) if n == 1 else ("strongly", "cross_mesh_2rot", "cross_mesh_cnot")):
        P = O.build_circuit(kind, n, L)[1]
        R = 37
        d = dict(a=rng.uniform(-0.9, 0.9, (R, n)), da=rng.normal(size=(3, R, n)),
                 qp=rng.uniform(0, 2 * np.pi, P), gz=rng.normal(size=(R, n)),
                 gdz=rng.normal(size=(3, R, n)))
        z, dz, zp, ga, gda, gq = _run(d, kind, "acos", L, dtype)
        wz, wdz = O.pqc_forward(d["a"], d["da"], d["qp"], kind, "acos", L)
        wga, wgda, wgq = O.pqc_backward(d["a"], d["da"], d["qp"], kind, "acos", L, d["gz"], d["gdz"])
        assert_close(z, wz, dtype, "z")
        assert_close(dz, wdz, dtype, "dz")
        assert_close(zp, wz, dtype, "zp")
        assert_close(ga, wga, dtype, "ga")
        assert_close(gda, wgda, dtype, "gda")
        assert_close(gq, wgq, dtype, "gq")


@pytest.mark.parametrize("dtype", DTYPES)
def test_pqc_large_batch_sampled_rows_and_properties(dtype):
    """R = 2^16 (config-2 size): sampled rows vs oracle, |<Z>| <= 1, and the
    no_entanglement/acos identity z == a at zero parameters (ansatz tests)."""
    from paper_2506_23246_b200.ansatz import build_circuit, pqc_forward_raw
    rng = np.random.default_rng(5)
    R, n, L = 1 << 16, 7, 4
    c = build_circuit("strongly", n, L)
    a = rng.uniform(-0.95, 0.95, (R, n))
    da = rng.normal(size=(3, R, n))
    qp = rng.uniform(0, 2 * np.pi, c.param_count)
    z, dz = pqc_forward_raw(c, "acos", cuda(a, dtype), cuda(da, dtype), cuda(qp, dtype))
    zc = z.double().cpu().numpy()
    assert np.all(np.abs(zc) <= 1 + 1e-5)
    idx = rng.choice(R, 64, replace=False)
    wz, wdz = O.pqc_forward(a[idx], da[:, idx], qp, "strongly", "acos", L)
    assert_close(z[idx], wz, dtype, "z sampled")
    assert_close(dz[:, idx], wdz, dtype, "dz sampled")
    c0 = build_circuit("no_entanglement", n, L)
    z0, _ = pqc_forward_raw(c0, "acos", cuda(a, dtype), None, cuda(np.zeros(c0.param_count), dtype))
    assert np.max(np.abs(z0.double().cpu().numpy() - a)) <= (1e-10 if dtype == torch.float64 else 2e-6)
    z1, _ = pqc_forward_raw(c0, "asin", cuda(a, dtype), None, cuda(np.zeros(c0.param_count), dtype))
    assert np.max(np.abs(z1.double().cpu().numpy() + a)) <= (1e-10 if dtype == torch.float64 else 2e-6)


def test_pqc_backward_is_bitwise_deterministic():
    from paper_2506_23246_b200.ansatz import build_circuit, pqc_backward_raw
    rng = np.random.default_rng(9)
    R, n = 20000, 7
    c = build_circuit("cross_mesh", n, 4)
    args = [cuda(x, torch.float32) for x in (rng.uniform(-0.9, 0.9, (R, n)), rng.normal(size=(3, R, n)),
                                              rng.uniform(0, 6, c.param_count), rng.normal(size=(R, n)),
                                              rng.normal(size=(3, R, n)))]
    r1 = pqc_backward_raw(c, "asin", *args)
    r2 = pqc_backward_raw(c, "asin", *args)
    for x, y in zip(r1, r2):
        assert torch.equal(x, y)


def test_quantum_layer_forward_autograd_and_domain():
    from paper_2506_23246_b200 import BatchedDual, DomainError, build_circuit, quantum_layer_forward
    rng = np.random.default_rng(2)
    c = build_circuit("strongly", 3, 2)
    d = golden_cases("pqc_small.npz")["strongly/acos"]
    a = cuda(d["a"], torch.float64).requires_grad_(True)
    da = cuda(d["da"], torch.float64).requires_grad_(True)
    qp = cuda(d["qp"], torch.float64).requires_grad_(True)
    out = quantum_layer_forward(BatchedDual(a, da), qp, c, "acos")
    loss = (out.val * cuda(d["gz"], torch.float64)).sum() + (out.tan * cuda(d["gdz"], torch.float64)).sum()
    loss.backward()
    assert_close(a.grad, d["ga"], torch.float64, "autograd g_a")
    assert_close(da.grad, d["gda"], torch.float64, "autograd g_da")
    assert_close(qp.grad, d["gq"], torch.float64, "autograd g_qp")
    bad = cuda(np.full((4, 3), 1.0 + 1e-9), torch.float64)
    with pytest.raises(DomainError):
        quantum_layer_forward(bad, qp.detach(), c, "acos")
    edge = cuda(np.full((4, 3), 1.0 + 5e-13), torch.float64)
    with pytest.warns(UserWarning):
        z = quantum_layer_forward(edge, qp.detach(), c, "acos")
    assert torch.isfinite(z).all()


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("kind", O.KINDS)
def test_specialized_kernels_match_generic_and_oracle(kind, dtype):
    """Compile-time specialised K1/K2 (GF(2) frame relabeling) vs the generic
    runtime-plan kernels and the oracle, with the state hand-off."""
    from paper_2506_23246_b200.ansatz import (build_circuit, pqc_backward_raw, pqc_forward_raw,
                                              state_buffer)
    rng = np.random.default_rng(11)
    n, L, R = 7, 4, 301
    res = {}
    for variant in ("layer", "generic", "auto"):
        c = build_circuit(kind, n, L)
        assert c.specialized
        c.set_kernel_variant(variant)
        d = dict(a=rng.uniform(-0.9, 0.9, (R, n)), da=rng.normal(size=(3, R, n)),
                 qp=rng.uniform(0, 2 * np.pi, c.param_count), gz=rng.normal(size=(R, n)),
                 gdz=rng.normal(size=(3, R, n))) if not res else res["d"]
        res["d"] = d
        a, da, qp = cuda(d["a"], dtype), cuda(d["da"], dtype), cuda(d["qp"], dtype)
        st = state_buffer(c, a)
        z, dz = pqc_forward_raw(c, "acos", a, da, qp, st)
        g = pqc_backward_raw(c, "acos", a, da, qp, cuda(d["gz"], dtype), cuda(d["gdz"], dtype), st)
        res[variant] = (z, dz) + g
    d = res["d"]
    wz, wdz = O.pqc_forward(d["a"], d["da"], d["qp"], kind, "acos", L)
    wg = O.pqc_backward(d["a"], d["da"], d["qp"], kind, "acos", L, d["gz"], d["gdz"])
    for variant in ("layer", "generic", "auto"):
        got = res[variant]
        for name, x, w in zip(("z", "dz", "ga", "gda", "gq"), got, (wz, wdz) + tuple(wg)):
            assert_close(x, w, dtype, f"{variant} {name}")


BIG_CASES = [(9, 2, "strongly", True), (10, 1, "cross_mesh_2rot", True), (11, 2, "cross_mesh", True),
             (9, 4, "cross_mesh", True), (10, 4, "strongly", True),
             (11, 2, "strongly", True), (12, 3, "cross_mesh", True),
             (12, 2, "strongly", True), (13, 1, "basic", True), (14, 1, "cross_mesh_cnot", True),
             (15, 1, "strongly", True), (16, 1, "no_entanglement", True),
             (16, 1, "cross_mesh", True), (15, 2, "cross_mesh_2rot", True)]


@pytest.mark.parametrize("n,L,kind,bwd", BIG_CASES)
def test_cluster_kernels_large_n_vs_oracle(n, L, kind, bwd):
    """n = 9..16 on the default dispatch vs the oracle: CTA / cluster kernels, the
    transfer map (n = 9, 10 from L = 4), and the multi-gate HBM passes (pqc_global.cu)
    where they take over -- including the mixed cases (n = 11 strongly, n = 12
    cross_mesh: forward on the CTA kernels, adjoint on the HBM passes)."""
    from paper_2506_23246_b200.ansatz import build_circuit, pqc_backward_raw, pqc_forward_raw
    dtype = torch.float32
    rng = np.random.default_rng(n * 7 + L)
    c = build_circuit(kind, n, L)
    R = 3
    d = dict(a=rng.uniform(-0.9, 0.9, (R, n)), da=rng.normal(size=(3, R, n)),
             qp=rng.uniform(0, 2 * np.pi, c.param_count), gz=rng.normal(size=(R, n)),
             gdz=rng.normal(size=(3, R, n)))
    a, da, qp = cuda(d["a"], dtype), cuda(d["da"], dtype), cuda(d["qp"], dtype)
    z, dz = pqc_forward_raw(c, "acos", a, da, qp)
    wz, wdz = O.pqc_forward(d["a"], d["da"], d["qp"], kind, "acos", L)
    # 3 points x up to 16 qubits: the per-tensor 1e-6 * max floor rests on a
    # handful of values, so n >= 13 is judged against the input-rounding floor
    fl = _floors(d, kind, "acos", L) if n >= 13 else [0.0] * 6
    assert_close_budget(z, wz, dtype, fl[0], f"n={n} z")
    assert_close_budget(dz, wdz, dtype, fl[1], f"n={n} dz")
    if bwd:
        ga, gda, gq = pqc_backward_raw(c, "acos", a, da, qp, cuda(d["gz"], dtype),
                                       cuda(d["gdz"], dtype))
        wga, wgda, wgq = O.pqc_backward(d["a"], d["da"], d["qp"], kind, "acos", L, d["gz"], d["gdz"])
        assert_close_budget(ga, wga, dtype, fl[3], f"n={n} ga")
        assert_close_budget(gda, wgda, dtype, fl[4], f"n={n} gda")
        assert_close_budget(gq, wgq, dtype, fl[5], f"n={n} gq")


@pytest.mark.parametrize("n,L,kind", [(9, 2, "strongly"), (10, 3, "cross_mesh"),
                                      (11, 2, "no_entanglement"), (12, 3, "strongly"),
                                      (12, 2, "cross_mesh_2rot"), (12, 2, "basic")])
def test_hbm_multigate_whole_state_tiles_vs_oracle(n, L, kind, monkeypatch):
    """The multi-gate HBM passes with one whole-state SM tile per row (n <= 12, no CS
    passes; the default for the n = 12 adjoint and CNOT-entangler forward) forced on
    from n = 9, K1 and K2 vs the oracle.  Every reverse pass holds the OUTER ops of
    one layer only (they read that layer's checkpoint)."""
    from paper_2506_23246_b200.ansatz import build_circuit, pqc_backward_raw, pqc_forward_raw
    monkeypatch.setenv("QPINN_PQC_HBM_FWD_MIN", "9")
    monkeypatch.setenv("QPINN_PQC_HBM_BWD_MIN", "9")
    dtype = torch.float32
    rng = np.random.default_rng(n * 17 + L)
    c = build_circuit(kind, n, L)
    R = 5
    d = dict(a=rng.uniform(-0.9, 0.9, (R, n)), da=rng.normal(size=(3, R, n)),
             qp=rng.uniform(0, 2 * np.pi, c.param_count), gz=rng.normal(size=(R, n)),
             gdz=rng.normal(size=(3, R, n)))
    a, da, qp = cuda(d["a"], dtype), cuda(d["da"], dtype), cuda(d["qp"], dtype)
    z, dz = pqc_forward_raw(c, "acos", a, da, qp)
    wz, wdz = O.pqc_forward(d["a"], d["da"], d["qp"], kind, "acos", L)
    fl = _floors(d, kind, "acos", L)
    assert_close_budget(z, wz, dtype, fl[0], f"n={n} z")
    assert_close_budget(dz, wdz, dtype, fl[1], f"n={n} dz")
    ga, gda, gq = pqc_backward_raw(c, "acos", a, da, qp, cuda(d["gz"], dtype),
                                   cuda(d["gdz"], dtype))
    wga, wgda, wgq = O.pqc_backward(d["a"], d["da"], d["qp"], kind, "acos", L, d["gz"], d["gdz"])
    assert_close_budget(ga, wga, dtype, fl[3], f"n={n} ga")
    assert_close_budget(gda, wgda, dtype, fl[4], f"n={n} gda")
    assert_close_budget(gq, wgq, dtype, fl[5], f"n={n} gq")


@pytest.mark.parametrize("n,L,kind", [(16, 1, "strongly"), (15, 1, "cross_mesh")])
def test_hbm_regime_adjoint_float64(n, L, kind):
    """float64 adjoint beyond the cluster-resident range vs the oracle (1e-10)."""
    from paper_2506_23246_b200.ansatz import build_circuit, pqc_backward_raw
    dtype = torch.float64
    rng = np.random.default_rng(n * 11 + L)
    c = build_circuit(kind, n, L)
    R = 2
    d = dict(a=rng.uniform(-0.9, 0.9, (R, n)), da=rng.normal(size=(3, R, n)),
             qp=rng.uniform(0, 2 * np.pi, c.param_count), gz=rng.normal(size=(R, n)),
             gdz=rng.normal(size=(3, R, n)))
    ga, gda, gq = pqc_backward_raw(c, "acos", cuda(d["a"], dtype), cuda(d["da"], dtype),
                                   cuda(d["qp"], dtype), cuda(d["gz"], dtype),
                                   cuda(d["gdz"], dtype))
    wga, wgda, wgq = O.pqc_backward(d["a"], d["da"], d["qp"], kind, "acos", L, d["gz"], d["gdz"])
    assert_close(ga, wga, dtype, f"n={n} ga")
    assert_close(gda, wgda, dtype, f"n={n} gda")
    assert_close(gq, wgq, dtype, f"n={n} gq")


@pytest.mark.parametrize("n,L,kind,dtype", [(9, 2, "strongly", torch.float32),
                                            (12, 1, "cross_mesh", torch.float64),
                                            (16, 1, "strongly", torch.float64),
                                            (15, 1, "cross_mesh_2rot", torch.float32)])
def test_global_memory_forward_vs_oracle(n, L, kind, dtype):
    """Value-only forward beyond the register kernels (any n) and the float64
    n = 16 forward with tangents run in global memory (pqc_global.cu)."""
    from paper_2506_23246_b200.ansatz import build_circuit, pqc_forward_raw
    rng = np.random.default_rng(n * 13 + L)
    c = build_circuit(kind, n, L)
    R = 3
    a = rng.uniform(-0.9, 0.9, (R, n))
    da = rng.normal(size=(3, R, n))
    qp = rng.uniform(0, 2 * np.pi, c.param_count)
    wz, wdz = O.pqc_forward(a, da, qp, kind, "acos", L)
    z, _ = pqc_forward_raw(c, "acos", cuda(a, dtype), None, cuda(qp, dtype))
    assert_close(z, wz, dtype, f"n={n} value-only z")
    if dtype == torch.float64 and n == 16:
        z, dz = pqc_forward_raw(c, "acos", cuda(a, dtype), cuda(da, dtype), cuda(qp, dtype))
        assert_close(z, wz, dtype, "z")
        assert_close(dz, wdz, dtype, "dz")


@pytest.mark.gpu
@pytest.mark.parametrize("R", [1000, 1, 65])
@pytest.mark.parametrize("n", [5, 6, 7, 8, 9, 10])
@pytest.mark.parametrize("kind", O.KINDS)
def test_transfer_matrix_kernels_vs_oracle(kind, n, R):
    """Transfer-matrix K1/K2 (variant "transfer": the circuit as one [2D, 2D]
    real map on the tensor cores, its adjoint on the D basis rows) vs the
    oracle, with and without the state hand-off, FP32 tolerance."""
    from paper_2506_23246_b200.ansatz import (build_circuit, pqc_backward_raw, pqc_forward_raw,
                                              state_buffer)
    if R != 1000 and kind not in ("strongly", "cross_mesh"):
        pytest.skip("ragged batch sizes: one permutation and one phase ansatz")
    if n == 10 and R == 1000:
        pytest.skip("n = 10: the ragged batches only (the oracle's 2^10 statevectors are slow)")
    dtype = torch.float32
    rng = np.random.default_rng(100 + n)
    L = 4
    c = build_circuit(kind, n, L)
    c.set_kernel_variant("transfer")
    d = dict(a=rng.uniform(-0.9, 0.9, (R, n)), da=rng.normal(size=(3, R, n)),
             qp=rng.uniform(0, 2 * np.pi, c.param_count), gz=rng.normal(size=(R, n)),
             gdz=rng.normal(size=(3, R, n)))
    a, da, qp = cuda(d["a"], dtype), cuda(d["da"], dtype), cuda(d["qp"], dtype)
    gz, gdz = cuda(d["gz"], dtype), cuda(d["gdz"], dtype)
    st = state_buffer(c, a)
    z, dz = pqc_forward_raw(c, "acos", a, da, qp, st)
    zp, _ = pqc_forward_raw(c, "acos", a, None, qp)
    g = pqc_backward_raw(c, "acos", a, da, qp, gz, gdz, st)
    g2 = pqc_backward_raw(c, "acos", a, da, qp, gz, gdz, None)
    wz, wdz = O.pqc_forward(d["a"], d["da"], d["qp"], kind, "acos", L)
    wg = O.pqc_backward(d["a"], d["da"], d["qp"], kind, "acos", L, d["gz"], d["gdz"])
    # a handful of points: the absolute floor (1e-6 of the largest entry) is taken over
    # only 7 .. 455 values, so small batches are judged against the input-rounding floor
    fl = _floors(d, kind, "acos", L) if R < 1000 else [0.0] * 6
    for name, x, w, f in zip(("z", "dz", "zp", "ga", "gda", "gq"), (z, dz, zp) + tuple(g),
                             (wz, wdz, wz) + tuple(wg), fl[:2] + fl[2:3] + fl[3:]):
        assert_close_budget(x, w, dtype, f, f"transfer {name}")
    for x, y in zip(g, g2):  # replayed forward: same launches, same bits
        assert torch.equal(x, y)


@pytest.mark.parametrize("dtype", DTYPES)
def test_torch_ops_boundary_default_7q_4l(dtype):
    """torch.ops.qpinn_b200.pqc_fwd_tangent / pqc_bwd_adjoint (SURVEY §8 b) with
    the K1 -> K2 state hand-off as a tensor, against the reference golden
    vectors, plus torch.library.opcheck of schema, fake and autograd
    registration."""
    from paper_2506_23246_b200.ansatz import build_circuit, plan_token
    for key, d in golden_cases("pqc_n7.npz").items():
        kind, scale = key.split("/")[:2]
        c = build_circuit(kind, 7, 4)
        tok = plan_token(c)
        a, da, qp = cuda(d["a"], dtype), cuda(d["da"], dtype), cuda(d["qp"], dtype)
        z, dz, st = torch.ops.qpinn_b200.pqc_fwd_tangent(tok, scale, a, da, qp, True)
        assert st.numel() > 0
        ga, gda, gq = torch.ops.qpinn_b200.pqc_bwd_adjoint(
            tok, scale, a, da, qp, st, cuda(d["gz"], dtype), cuda(d["gdz"], dtype))
        assert_close(z, d["z"], dtype, f"{key} z")
        assert_close(dz, d["dz"], dtype, f"{key} dz")
        assert_close(ga, d["ga"], dtype, f"{key} g_a")
        assert_close(gda, d["gda"], dtype, f"{key} g_da")
        assert_close(gq, d["gq"], dtype, f"{key} g_qparams")
    torch.library.opcheck(torch.ops.qpinn_b200.pqc_fwd_tangent.default,
                          (tok, scale, a, da, qp, True),
                          test_utils=("test_schema", "test_faketensor",
                                      "test_autograd_registration"))


def test_transfer_forward_repeatable_under_load():
    """The transfer-path forward (tensor-core map + fused readout, and the
    value-only map + readout pass) is bitwise repeatable over many launches."""
    from paper_2506_23246_b200.ansatz import build_circuit, pqc_forward_raw
    rng = np.random.default_rng(11)
    R, n = 1 << 16, 7
    c = build_circuit("strongly", n, 4)
    a = cuda(rng.uniform(-0.95, 0.95, (R, n)), torch.float32)
    da = cuda(rng.normal(size=(3, R, n)), torch.float32)
    qp = cuda(rng.uniform(0, 2 * np.pi, c.param_count), torch.float32)
    for tan in (da, None):
        z0, dz0 = pqc_forward_raw(c, "acos", a, tan, qp)
        for _ in range(60):
            z, dz = pqc_forward_raw(c, "acos", a, tan, qp)
            assert torch.equal(z, z0)
            if tan is not None:
                assert torch.equal(dz, dz0)


@pytest.mark.parametrize("n", [4, 7])
def test_parameter_shift_matches_adjoint_f64(n):
    """The reference suite's shift-rule check (test_qsim.py:139-166) on our kernels:
    d(sum z)/d(theta) from two shifted K1 launches per slot equals K2's adjoint
    gradient to 1e-10 in fp64 (strongly: every slot in a single-axis rotation)."""
    from paper_2506_23246_b200.ansatz import build_circuit, pqc_backward_raw, pqc_forward_raw
    rng = np.random.default_rng(21)
    L, R = 2, 16
    c = build_circuit("strongly", n, L)
    a = cuda(rng.uniform(-0.9, 0.9, (R, n)), torch.float64)
    da = cuda(np.zeros((3, R, n)), torch.float64)
    qp0 = rng.uniform(0, 2 * np.pi, c.param_count)
    gz = cuda(np.ones((R, n)), torch.float64)
    _, _, gq = pqc_backward_raw(c, "acos", a, da, cuda(qp0, torch.float64), gz,
                                cuda(np.zeros((3, R, n)), torch.float64))

    def f(q):
        return pqc_forward_raw(c, "acos", a, da, cuda(q, torch.float64))[0].sum().item()

    shift = np.array([(f(qp0 + np.pi / 2 * e) - f(qp0 - np.pi / 2 * e)) / 2.0
                      for e in np.eye(qp0.size)])
    assert np.max(np.abs(shift - gq.cpu().numpy())) <= 1e-10


@pytest.mark.parametrize("kind,n", [("cross_mesh", 5), ("strongly", 7), ("basic", 10)])
def test_tangents_match_central_differences_f64(kind, n):
    """K1's forward-mode tangents against central differences of its own values
    (test_autodiff.py:129-150 on our kernels), fp64."""
    from paper_2506_23246_b200.ansatz import build_circuit, pqc_forward_raw
    rng = np.random.default_rng(22)
    L, R = 3, 12
    c = build_circuit(kind, n, L)
    a = rng.uniform(-0.8, 0.8, (R, n))
    da = rng.normal(size=(3, R, n))
    qp = cuda(rng.uniform(0, 2 * np.pi, c.param_count), torch.float64)
    _, dz = pqc_forward_raw(c, "asin", cuda(a, torch.float64), cuda(da, torch.float64), qp)
    h = 1e-6
    for k in range(3):
        zp = pqc_forward_raw(c, "asin", cuda(a + h * da[k], torch.float64), None, qp)[0]
        zm = pqc_forward_raw(c, "asin", cuda(a - h * da[k], torch.float64), None, qp)[0]
        fd = ((zp - zm) / (2 * h)).cpu().numpy()
        assert np.max(np.abs(fd - dz[k].cpu().numpy())) <= 1e-7
