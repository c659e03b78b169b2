"""Full train-step parity on the GPU: LossEvaluator.evaluate(tape=True)
gradients/breakdowns vs reference golden vectors, and loss curves vs the
reference trainer."""
import numpy as np
import pytest
import torch

from conftest import load_golden
from gpu_util import assert_close, norm_rel

pytestmark = pytest.mark.gpu


def _build(g, dtype):
    from paper_2506_23246_b200.network import Model, ModelConfig
    from paper_2506_23246_b200.physics import CollocationGrid, LossEvaluator, MaterialMap
    h, F, n, L, seed = (int(v) for v in g["config"])
    cfg = ModelConfig(variant="hybrid", hidden_width=h, rff_features=F, n_qubits=n,
                      n_layers_pqc=L, ansatz=str(g["ansatz"]), scale=str(g["scale"]), seed=seed,
                      t_domain=float(g["t_domain"]))
    model = Model(cfg, device="cuda", dtype=dtype)
    grid = CollocationGrid(*(int(v) for v in g["grid"]), float(g["t_end"]))
    case = str(g["case"])
    ev = LossEvaluator(model, grid, MaterialMap(case), case=case, phys_mode=str(g["phys_mode"]),
                       energy_enabled=bool(g["energy"]), chunk_slices=int(g["chunk_slices"]))
    return model, ev


def _check_grad(got, want, dtype, what):
    """float64: 1e-10 elementwise; float32: the flat gradient (66,932 entries,
    many at rounding level) within 1e-5 norm-relative (north_star's 1e-5 on
    the vector)."""
    if dtype == torch.float64:
        assert_close(got, want, dtype, what)
    else:
        e = norm_rel(got, want)
        assert e <= 1e-5, f"{what}: norm-relative {e:.3e}"


def _check_fields(got, want, dtype, what):
    """Model outputs through the whole chain (trunk, PQC, head): float64
    elementwise 1e-10; float32 norm-relative 1e-5 (SURVEY 8.C's alternative
    definition; elementwise errors and their input-rounding floors are in
    profiles/r02/fp32_error_budget.json)."""
    if dtype == torch.float64:
        assert_close(got, want, dtype, what)
    else:
        e = norm_rel(got, want)
        assert e <= 1e-5, f"{what}: norm-relative {e:.3e}"


EVALS = ["eval_micro_vacuum.npz", "eval_micro_diel.npz", "eval_micro_asym.npz", "eval_desk.npz",
         "eval_vacuum7.npz", "eval_diel7.npz",
         # 6 qubits: the transfer-matrix PQC kernels (permutation and phase entanglers)
         "eval_n6_strongly.npz", "eval_n6_crossmesh.npz",
         # 8 and 9 qubits: the transfer map where it became the default in round 2
         "eval_n8_strongly.npz", "eval_n9_crossmesh.npz", "eval_n10_2rot.npz",
         # 12 qubits: the multi-gate HBM passes (K1 and K2)
         "eval_n12_strongly.npz"]


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("name", EVALS)
def test_evaluate_tape_matches_reference(name, dtype):
    g = load_golden(name)
    model, ev = _build(g, dtype)
    params = model.params_from(g["flat"])
    assert np.array_equal(model.init_params_np(), g["flat"])
    w = g["weights"] if g["weights"].size else None
    res = ev.evaluate(params, weights=w, tape=True)
    bd = res.breakdown
    got = np.array([bd.phys, bd.ic, bd.sym, bd.energy, bd.total])
    assert_close(got, g["breakdown"], dtype, "breakdown")
    assert_close(np.array(bd.bin_phys), g["bin_phys"], dtype, "bin_phys")
    _check_grad(res.grad, g["grad"], dtype, "flat gradient")
    from paper_2506_23246_b200.network import FieldBatch
    x, y, t = ev.grid.flat_points()
    fields, derivs = model.forward(params, x, y, t, derivs=True)
    _check_fields(torch.stack([fields.ez, fields.hx, fields.hy]), g["fields"], dtype, "fields")
    _check_fields(torch.stack([derivs.ez, derivs.hx, derivs.hy]), g["derivs"], dtype, "derivs")
    # independent cross-check: torch-autograd trunk + K1/K2/K4 autograd functions
    ref = ev.evaluate(params, weights=w, tape=True, native=False)
    _check_grad(ref.grad, g["grad"], dtype, "autograd-path gradient")
    plain = ev.evaluate(params, weights=w, tape=False)
    assert abs(plain.breakdown.total - float(g["plain_total"])) <= (1e-10 if dtype == torch.float64 else 1e-4) * abs(float(g["plain_total"]))


@pytest.mark.parametrize("dtype,epochs,rtol", [(torch.float64, 1000, 1e-9), (torch.float32, 1000, 1e-4)])
def test_train_curve_matches_reference_desk(dtype, epochs, rtol):
    """1k Adam steps of the desk_smoke model (4q x 2L, 8x8x10 grid)."""
    from paper_2506_23246_b200.network import ModelConfig
    from paper_2506_23246_b200.training import TrainConfig, train
    g = load_golden("train_desk.npz")
    h, F, n, L, seed = (int(v) for v in g["config"])
    cfg = TrainConfig(case="vacuum", model=ModelConfig(variant="hybrid", hidden_width=h,
                      rff_features=F, n_qubits=n, n_layers_pqc=L, ansatz=str(g["ansatz"]),
                      scale=str(g["scale"]), seed=seed), epochs=epochs,
                      grid=tuple(int(v) for v in g["grid"]), eval_cadence=0, probe_cadence=0)
    res = train(cfg, dtype=dtype)
    tot = np.array([r.total for r in res.log.rows])
    want = g["total"][:epochs]
    rel = np.max(np.abs(tot - want) / np.abs(want))
    assert rel <= rtol, rel


def test_train_curve_matches_reference_vacuum7_fp64():
    """Full-width 7q x 4L model (66,932 params), 200 epochs on a 4x4x6 grid."""
    from paper_2506_23246_b200.network import ModelConfig
    from paper_2506_23246_b200.training import TrainConfig, train
    g = load_golden("train_vacuum7.npz")
    cfg = TrainConfig(case="vacuum", model=ModelConfig(variant="hybrid", ansatz="strongly",
                      scale="acos", seed=0), epochs=200, grid=(4, 4, 6), eval_cadence=0,
                      probe_cadence=0)
    res = train(cfg, dtype=torch.float64)
    tot = np.array([r.total for r in res.log.rows])
    rel = np.max(np.abs(tot - g["total"]) / np.abs(g["total"]))
    assert rel <= 1e-8, rel
    assert np.allclose(res.params.flat.cpu().numpy(), g["final_flat"], rtol=1e-7, atol=1e-9)


@pytest.mark.parametrize("host_inputs", [False, True])
def test_cuda_graph_steps_match_eager_bitwise(host_inputs):
    """The replayed CUDA graph of the step's device part (several chunks,
    alternating bin-weight buffers, optional pinned-host input copies) gives
    bit-identical losses and parameters to eager launches."""
    from paper_2506_23246_b200.network import ModelConfig
    from paper_2506_23246_b200.training import TrainConfig, Trainer
    cfg = TrainConfig(case="vacuum", model=ModelConfig(variant="hybrid", ansatz="strongly",
                      scale="acos", seed=0), epochs=6, grid=(16, 16, 12), chunk_slices=4,
                      eval_cadence=0, probe_cadence=0)
    runs = []
    for graphs in (False, True):
        tr = Trainer(cfg, device="cuda", dtype=torch.float32, graphs=graphs)
        tr.set_host_inputs(host_inputs)
        rows = [tr.step().total for _ in range(6)]
        runs.append((rows, tr.flat.detach().cpu().numpy().copy()))
        if graphs:
            assert tr._graphs, "no graph was captured"
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])
