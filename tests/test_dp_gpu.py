"""Data-parallel Trainer end to end on the real engine: two ranks (gloo for
the one all-reduce, host-staged) sharing one GPU.  The ranks' kernels never
wait on each other -- the only exchange is the host-side collective between
the graph-replayed local sweeps -- and the result must equal one rank doing
the whole grid (sharding whole time slices is exact; float64,
so only the summation order differs)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _cfg():
    from paper_2506_23246_b200.network import ModelConfig
    from paper_2506_23246_b200.training import TrainConfig
    return TrainConfig(case="vacuum", model=ModelConfig(variant="hybrid", ansatz="strongly",
                       scale="acos", seed=0, hidden_width=32, rff_features=16),
                       epochs=4, grid=(8, 8, 10), chunk_slices=2, eval_cadence=0,
                       probe_cadence=0)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_23246_b200.training import Trainer

    def host_allreduce(t):
        c = t.cpu()
        dist.all_reduce(c)
        t.copy_(c)

    tr = Trainer(_cfg(), device="cuda:0", dtype=torch.float64, rank=rank, world_size=world,
                 reduce_fn=host_allreduce)
    totals = [tr.step().total for _ in range(4)]
    out[rank] = (totals, tr.flat.detach().cpu().numpy().copy(), bool(tr._graphs))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_match_single_rank():
    from paper_2506_23246_b200.training import Trainer
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    one = Trainer(_cfg(), device="cuda:0", dtype=torch.float64)
    totals = [one.step().total for _ in range(4)]
    flat = one.flat.detach().cpu().numpy()
    for r in range(2):
        t_r, f_r, graphed = out[r]
        assert graphed, "the local sweep should replay from a CUDA graph"
        assert np.allclose(t_r, totals, rtol=1e-12, atol=0)
        # Adam normalises each gradient entry by its own running magnitude, so
        # entries whose gradient is at rounding level can move by O(lr) eps
        # differently; everything else agrees to float64 rounding
        d = np.abs(f_r - flat)
        assert np.max(d) <= 1e-9, np.max(d)
        assert np.mean(d <= 1e-13 * np.maximum(np.abs(flat), 1.0)) > 0.99
    assert np.array_equal(out[0][1], out[1][1])  # replicated Adam: identical parameters


def _domain_worker(rank, world, port, out):
    """The real engine on two ranks: rank 1's PQC forward folds max|a| = 1.5
    (written into its running maximum, as a kernel excursion would be) -> the
    domain flags travel in the step's one all-reduce, Adam is vetoed on the
    device and both ranks raise DomainError with their parameters untouched."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_23246_b200.errors import DomainError
    from paper_2506_23246_b200.training import Trainer

    def host_allreduce(t):
        c = t.cpu()
        dist.all_reduce(c)
        t.copy_(c)

    tr = Trainer(_cfg(), device="cuda:0", dtype=torch.float32, rank=rank, world_size=world,
                 reduce_fn=host_allreduce)
    tr.step()
    before = tr.flat.detach().cpu().numpy().copy()
    t_before = tr.adam.t
    if rank == 1:
        tr._pqc_workspace()[:8].copy_(
            torch.tensor([1.5], dtype=torch.float64).view(torch.uint8).to("cuda:0"))
    try:
        tr.step()
        out[rank] = "no error"
    except DomainError as e:
        out[rank] = "DomainError: " + str(e)
    out[f"same{rank}"] = bool(np.array_equal(before, tr.flat.detach().cpu().numpy())) and \
        tr.adam.t == t_before
    dist.barrier()
    dist.destroy_process_group()


def test_domain_error_on_rank1_raises_on_both_ranks():
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_domain_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    for r in range(2):
        assert out[r].startswith("DomainError"), out[r]
        assert out[f"same{r}"], "Adam must be vetoed: parameters and step count unchanged"
