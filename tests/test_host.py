"""Host-side logic that needs no GPU: grid/bin/normaliser tables, parameter
layout + RNG streams, data-parallel sharding arithmetic."""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import load_golden


def test_model_layout_and_init_match_reference_golden():
    from paper_2506_23246_b200.network import Model, ModelConfig
    g = load_golden("eval_vacuum7.npz")
    m = Model(ModelConfig(variant="hybrid", ansatz="strongly", scale="acos", seed=0),
              device="cpu", dtype=torch.float64)
    assert m.total_parameter_count == 66932
    names = [(n, o) for n, o, _ in m.layout]
    assert names[-1] == ("quantum", 66848)
    assert dict(names)["tau_raw"] == 66847
    assert np.array_equal(m.init_params_np(), g["flat"])


def test_shard_slices_partition():
    from paper_2506_23246_b200.training import shard_slices
    for nt in (1, 5, 16, 64, 67):
        for world in (1, 2, 3, 4, 8):
            parts = [shard_slices(nt, r, world) for r in range(world)]
            flat = [s for p in parts for s in p]
            assert flat == list(range(nt))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1


def test_time_bin_weights_matches_oracle(rng):
    from paper_2506_23246_b200.physics import time_bin_weights
    for _ in range(20):
        b = rng.uniform(0, 3, 5)
        assert np.allclose(time_bin_weights(b, 1.3), O.time_bin_weights(b, 1.3), rtol=0, atol=0)


def test_grid_bins_and_mirrors_match_oracle():
    from paper_2506_23246_b200.physics import CollocationGrid
    for dims in ((64, 64, 16), (128, 128, 64), (6, 4, 5)):
        g = CollocationGrid(*dims, 1.5)
        o = O.Grid(*dims, 1.5)
        assert [g.bin_of_slice(i) for i in range(g.nt)] == [o.bin_of_slice(i) for i in range(o.nt)]
        assert np.array_equal(g.mirror_x_local, o.mirror_x)
        assert np.array_equal(g.mirror_y_local, o.mirror_y)
    g = CollocationGrid(64, 64, 16, 1.5)
    pops = [sum(1 for i in range(16) if g.bin_of_slice(i) == m) for m in range(5)]
    assert pops == [3, 3, 3, 3, 4]


def test_torch_ops_registered_with_shapes():
    """The custom-op boundary (SURVEY §8 b) is registered and shape-infers on
    meta tensors without a GPU (no compute)."""
    import torch
    from paper_2506_23246_b200.ansatz import build_circuit, plan_token
    c = build_circuit("cross_mesh", 7, 4)
    a = torch.empty(10, 7, device="meta")
    da = torch.empty(3, 10, 7, device="meta")
    qp = torch.empty(c.param_count, device="meta")
    z, dz, st = torch.ops.qpinn_b200.pqc_fwd_tangent(plan_token(c), "acos", a, da, qp, True)
    assert z.shape == (10, 7) and dz.shape == (3, 10, 7) and st.numel() > 0
    _, _, st0 = torch.ops.qpinn_b200.pqc_fwd_tangent(plan_token(c), "acos", a, da, qp, False)
    assert st0.numel() == 0
    ga, gda, gq = torch.ops.qpinn_b200.pqc_bwd_adjoint(plan_token(c), "acos", a, da, qp, st, z, dz)
    assert ga.shape == (10, 7) and gda.shape == (3, 10, 7) and gq.shape == (c.param_count,)


def test_embedding_phase_folding_identity():
    """The transfer path's phase folding (csrc/pqc_transfer.cu tr_wmat / tr_gb):
    every embedded row is phi_b = (-i)^popcount(b) m_b with real m_b, so the
    real-block map [Re phi | Im phi] W equals m W' with W' = Re p W[:D] + Im p W[D:],
    and dL/dW is recovered from dL/dW' = m^T Abar row by row."""
    import numpy as np
    rng = np.random.default_rng(3)
    n, R = 5, 9
    D = 1 << n
    B = rng.normal(size=(D, D)) + 1j * rng.normal(size=(D, D))
    W = np.block([[B.real, B.imag], [-B.imag, B.real]])
    p = (-1j) ** np.array([bin(b).count("1") for b in range(D)])
    m = rng.normal(size=(R, D))
    phi = m * p
    Phi = np.concatenate([phi.real, phi.imag], axis=1)
    Wf = p.real[:, None] * W[:D] + p.imag[:, None] * W[D:]
    np.testing.assert_allclose(Phi @ W, m @ Wf, rtol=0, atol=1e-12)
    Abar = rng.normal(size=(R, 2 * D))
    # dL/dm is the phase-aligned projection of dL/dPhi
    gPhi = Abar @ W.T
    np.testing.assert_allclose(Abar @ Wf.T, p.real * gPhi[:, :D] + p.imag * gPhi[:, D:], atol=1e-12)
    gW = Phi.T @ Abar
    gWf = m.T @ Abar
    np.testing.assert_allclose(gW[:D], p.real[:, None] * gWf, atol=1e-12)
    np.testing.assert_allclose(gW[D:], p.imag[:, None] * gWf, atol=1e-12)
