"""Row-wise sharding on the B200 engine (key placement by the
reference store's fnv1a64(table, row) mod N, store.py:80-88): every shard of
a Criteo-like trace run by the pipelined engine (one after the other on one
GPU -- the shards share nothing), the union of the written rows equals the
unsharded run's store bit for bit, and each shard's writes are exactly the
keys it owns.  Also the occurrence-backed batches of a row shard through the
generic prep: same plan stream as the CPU oracle."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import bagpipe_oracle as O
from paper_2202_12429_b200.traces import Schema, ZipfSpec, batchify_columns, generate_columns

pytestmark = pytest.mark.gpu

SCHEMA = Schema(5, (3, 70_000, 1_000, 400_000, 17), 2, 8)


def _trace(n_batches=10, batch=2048, seed=21):
    rows, labels, dense = generate_columns(ZipfSpec(SCHEMA, 1.05, n_batches * batch, seed))
    return batchify_columns(rows, labels, dense, batch)


def _written(report) -> dict:
    return {(k[0] << 44) | k[1]: v for k, v in report.final_store.written_items()}


@pytest.mark.parametrize("world,trainers", [(2, 2), (3, 1), (4, 4)])
def test_row_shards_union_equals_unsharded_run(world, trainers):
    from paper_2202_12429_b200.engine import EngineConfig, run_pipeline
    from paper_2202_12429_b200.shard import row_owner, row_shard_batches

    batches = _trace()
    cfg = EngineConfig(cache_capacity=40_000, batch_size=2048, lookahead=4, num_trainers=trainers, num_shards=1,
                       seed=7)
    want = _written(run_pipeline(cfg, SCHEMA, batches))
    merged = {}
    for rank in range(world):
        got = _written(run_pipeline(cfg, SCHEMA, row_shard_batches(batches, world, rank)))
        keys = np.fromiter(got.keys(), dtype=np.uint64, count=len(got))
        assert np.all(row_owner(keys, world) == rank)
        assert not (set(got) & set(merged))
        merged.update(got)
    assert set(merged) == set(want)
    for k, v in want.items():
        np.testing.assert_array_equal(merged[k], v)


def test_row_shard_plan_stream_matches_oracle():
    from paper_2202_12429_b200 import lookahead as lk
    from paper_2202_12429_b200.shard import row_shard_batches

    shard = row_shard_batches(_trace(6, 1024, seed=5), 3, 1)
    want = [O.plan_sha(p) for p in O.plan_stream(shard, 3, 20_000)[0]]
    state = lk.new_state(3, 20_000, schema=SCHEMA)
    src = iter(shard)
    got = []
    while (p := lk.emit_next_plan(state, src)) is not None:
        pf = O.pack([k[0] for k in p.prefetch], [k[1] for k in p.prefetch]) if p.prefetch else []
        uniq = O.pack([k[0] for k, _ in p.ttl_updates], [k[1] for k, _ in p.ttl_updates])
        got.append(O.plan_sha((p.iteration, pf, uniq, [t for _, t in p.ttl_updates], None, p.lookahead)))
        lk.adapt_on_pressure(state)
    assert got == want
