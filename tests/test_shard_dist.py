"""N>1 host logic on CPU with gloo (world_size 2 and 3): table-wise and
row-wise (fnv1a64 key placement, reference store.py:80-88) shards of the
pipelined path, each run by the CPU oracle on its rank, gathered to rank 0,
reproduce the unsharded final store bit for bit."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import pytest

from paper_2202_12429_b200.shard import row_shard_batches, shard_batches, table_shards
from paper_2202_12429_b200.traces import Schema, ZipfSpec, batchify_columns, generate_columns

SCHEMA = Schema(3, (600, 400, 50), 2, 4)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _trace():
    rows, labels, dense = generate_columns(ZipfSpec(SCHEMA, 1.05, 40 * 64, seed=11))
    return batchify_columns(rows, labels, dense, 64)


def _rank_main(rank, world, port, out, mode="table"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import bagpipe_oracle as O

    if mode == "table":
        mine = shard_batches(_trace(), table_shards(SCHEMA.num_tables, world)[rank])
    else:
        mine = row_shard_batches(_trace(), world, rank)
    store, _ = O.pipeline(mine, SCHEMA.rows_per_table, 4, 5, 2, 10_000, 6, 0.25)
    gathered = [None] * world
    dist.all_gather_object(gathered, store.values)
    t = torch.tensor([float(rank + 1)])  # the bench's timing reduction: max over ranks
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        merged = {}
        for part in gathered:
            assert not (set(part) & set(merged)), "shards own disjoint keys"
            merged.update(part)
        out.put((merged, float(t)))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,world", [("table", 2), ("row", 2), ("row", 3)])
def test_sharding_is_exact_with_gloo(mode, world):
    from oracle import bagpipe_oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    merged, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == float(world)
    store, _ = O.pipeline(_trace(), SCHEMA.rows_per_table, 4, 5, 2, 10_000, 6, 0.25)
    assert set(merged) == set(store.values)
    for k, v in store.values.items():
        assert np.array_equal(merged[k], v)
    rebuilt = O.Store(SCHEMA.rows_per_table, 4, 5)
    rebuilt.values = merged
    assert rebuilt.digest() == store.digest()
