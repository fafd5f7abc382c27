"""DLRM hybrid parallelism host logic on CPU ranks (gloo): model-parallel
embedding tables (round-robin shards) + data-parallel MLP, with the
EmbeddingExchange all-to-alls and the mean all-reduce, trains exactly like
one process on the whole batch (fp64, so only summation order differs)."""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2202_12429_b200.dlrm import DLRMDense
from paper_2202_12429_b200.hybrid import EmbeddingExchange, allreduce_mean_

T, D, ROWS, B, NDENSE, STEPS = 5, 4, 7, 12, 3, 3


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(step):
    g = torch.Generator().manual_seed(100 + step)
    idx = torch.randint(0, ROWS, (B, T), generator=g)
    dense = torch.randn(B, NDENSE, generator=g, dtype=torch.float64)
    labels = (torch.rand(B, generator=g) > 0.5).double()
    return idx, dense, labels


def _init():
    torch.manual_seed(0)
    model = DLRMDense(NDENSE, T, D, bottom=(8,), top=(8,)).double()
    tables = [torch.randn(ROWS, D, dtype=torch.float64) for _ in range(T)]
    return model, tables


def _single(lr):
    model, tables = _init()
    tables = [t.clone().requires_grad_(True) for t in tables]
    opt = torch.optim.SGD(list(model.parameters()) + tables, lr=lr)
    for step in range(STEPS):
        idx, dense, labels = _data(step)
        emb = torch.stack([tables[t][idx[:, t]] for t in range(T)], 1)
        loss = torch.nn.functional.binary_cross_entropy_with_logits(model(dense, emb), labels)
        opt.zero_grad()
        loss.backward()
        opt.step()
    return model, [t.detach() for t in tables]


def _rank_main(rank, world, port, lr, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model, tables = _init()
    ex = EmbeddingExchange(T, D, rank, world)
    mine = {t: tables[t].clone().requires_grad_(True) for t in ex.local_tables}
    mopt = torch.optim.SGD(model.parameters(), lr=lr)
    eopt = torch.optim.SGD(list(mine.values()), lr=lr)
    bl = B // world
    for step in range(STEPS):
        idx, dense, labels = _data(step)
        pooled_local = torch.stack([mine[t][idx[:, t]] for t in ex.local_tables], 1)   # [B, T_r, D]
        emb = ex.forward(pooled_local.detach()).requires_grad_(True)                  # [B/N, T, D]
        sl = slice(rank * bl, (rank + 1) * bl)
        loss = torch.nn.functional.binary_cross_entropy_with_logits(model(dense[sl], emb), labels[sl])
        mopt.zero_grad()
        eopt.zero_grad()
        loss.backward()
        allreduce_mean_([p.grad for p in model.parameters()], world)
        pooled_local.backward(ex.backward(emb.grad, scale=1.0 / world))
        mopt.step()
        eopt.step()
    # numpy (pickled by value): torch tensors would travel as shared-memory fds
    out.put((rank, {t: v.detach().numpy().copy() for t, v in mine.items()},
             {k: v.numpy().copy() for k, v in model.state_dict().items()}))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_hybrid_dlrm_equals_single_process(world):
    lr = 0.1
    want_model, want_tables = _single(lr)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, lr, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    seen = set()
    for rank, mine, state in results:
        for t, v in mine.items():
            torch.testing.assert_close(torch.from_numpy(v), want_tables[t], rtol=1e-12, atol=1e-12)
            seen.add(t)
        for name, v in want_model.state_dict().items():
            torch.testing.assert_close(torch.from_numpy(state[name]), v, rtol=1e-12, atol=1e-12, msg=name)
    assert seen == set(range(T))
