"""Data-parallel host path on CPU with the gloo backend (world_size 2 and 3).

Each rank evaluates its contiguous block of whole time slices (here with the
numpy oracle standing in for the device sweep, which needs a GPU), packs
[gradient | 23 loss sums] exactly as the Trainer does, all-reduces once, and
the result must equal the single-process full-grid evaluation (SURVEY 8e:
sharding whole slices is exact)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O

KEY_SLOT = {"res1": 0, "res1_vac": 0, "res1_diel": 1, "res2": 2, "res3": 3}


def _pack_sums(bin_sums, sums):
    v = np.zeros(23)
    for m, d in enumerate(bin_sums):
        for k, val in d.items():
            v[4 * m + KEY_SLOT[k]] += val
    v[20], v[21], v[22] = sums["energy"], sums["sym"], sums["ic"]
    return v


def _setup(case):
    model = O.OracleModel(hidden=6, rff=5, n_qubits=3, n_layers=2, ansatz="cross_mesh",
                          scale="asin", seed=5, t_domain=1.5 if case != "dielectric" else 0.7)
    grid = O.Grid(6, 4, 7, model.t_domain)
    return model, grid


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_23246_b200.training import allreduce_fn, reduce_packed, shard_slices
    model, grid = _setup(case)
    flat = model.init_params()
    w = np.array([1.0, 0.7, 0.5, 0.3, 0.2])
    ev = O.Evaluator(model, grid, case=case, chunk_slices=2,
                     slices=shard_slices(grid.nt, rank, world))
    _, grad, (bin_sums, sums) = ev.evaluate(flat, w, tape=True)
    g = torch.tensor(grad, dtype=torch.float32)
    s = torch.tensor(_pack_sums(bin_sums, sums), dtype=torch.float64)
    reduce_packed(g, s, allreduce_fn())
    out[rank] = (g.numpy().copy(), s.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,case", [(2, "vacuum"), (3, "dielectric")])
def test_dp_allreduce_matches_full_grid(world, case):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    model, grid = _setup(case)
    w = np.array([1.0, 0.7, 0.5, 0.3, 0.2])
    full_bd, full_grad, (bin_sums, sums) = O.Evaluator(model, grid, case=case,
                                                       chunk_slices=2).evaluate(
        model.init_params(), w, tape=True)
    full_sums = _pack_sums(bin_sums, sums)
    for r in range(world):
        g, s = out[r]
        # every rank holds the same reduced vector
        assert np.array_equal(g, out[0][0]) and np.array_equal(s, out[0][1])
        # gradient reduced in float64 then cast: float32 rounding only
        assert np.allclose(g, full_grad, rtol=1e-6, atol=1e-7 * np.abs(full_grad).max())
        assert np.allclose(s, full_sums, rtol=1e-12, atol=1e-15)


def test_shard_evaluators_cover_grid_once():
    model, grid = _setup("vacuum")
    seen = []
    from paper_2506_23246_b200.training import shard_slices
    for r in range(4):
        ev = O.Evaluator(model, grid, chunk_slices=2, slices=shard_slices(grid.nt, r, 4))
        for _, sl in ev.chunks:
            seen += list(sl)
    assert sorted(seen) == list(range(grid.nt))


def _domain_worker(rank, world, port, out):
    """Rank 1 alone sees |a| > 1 + 1e-12: the flags ride in the packed
    all-reduce, so every rank raises DomainError (none is left blocked in the
    next collective)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_23246_b200.errors import DomainError
    from paper_2506_23246_b200.training import allreduce_fn, raise_domain, reduce_packed
    grad = torch.full((5,), float(rank), dtype=torch.float32)
    sums = torch.zeros(23, dtype=torch.float64)
    dom = torch.tensor([1.0, 1.0, 1.5] if rank == 1 else [0.0, 0.0, 0.7], dtype=torch.float64)
    reduce_packed(grad, sums, allreduce_fn(), extra=dom[:2])
    try:
        raise_domain(*dom.tolist())
        out[rank] = "no error"
    except DomainError as e:
        out[rank] = "DomainError: " + str(e)
    # the process group is still usable by every rank afterwards
    t = torch.ones(1)
    dist.all_reduce(t)
    out[f"after{rank}"] = float(t)
    dist.destroy_process_group()


def test_domain_error_on_one_rank_raises_on_every_rank():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_domain_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        assert out[r].startswith("DomainError"), out[r]
        assert out[f"after{r}"] == 2.0


def test_clamp_flag_warns_without_error():
    from paper_2506_23246_b200.training import raise_domain
    with pytest.warns(UserWarning, match="clamped"):
        raise_domain(0.0, 1.0, 1.0 + 1e-13)
    raise_domain(0.0, 0.0, 0.9)
