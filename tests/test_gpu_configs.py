"""SURVEY 8(d) configurations 3-5 as parity cases (reduced batch counts so
the CPU oracle finishes in seconds): Avazu W&D shape (22 tables, ~9.4M rows),
a Terabyte-like shape at D=64, and sweep cells over window x cache x Zipf,
including cells where the capacity is exceeded -- which must fail at the
same iteration on both sides.  Checks: pipelined == synchronous baseline
digests, and every written store row equal to the oracle's."""

from __future__ import annotations

import re

import numpy as np
import pytest

from oracle import bagpipe_oracle as O
from paper_2202_12429_b200.traces import Schema, ZipfSpec, batchify_columns, generate_columns

pytestmark = pytest.mark.gpu

# 22 categorical columns summing to 9,449,206 rows ("9.4M
# embeddings"; the reference ships no Avazu cardinalities, this split is ours)
AVAZU_ROWS = (7, 7, 4737, 7745, 26, 8552, 559, 36, 2686408, 6729486, 8251, 5, 4, 2626, 8, 9, 435, 4, 68, 172,
              60, 1)


def _engine():
    from paper_2202_12429_b200 import engine

    return engine


def _run_and_compare(schema, batches, cfg):
    eng = _engine()
    pipe = eng.run_pipeline(cfg, schema, batches)
    base = eng.run_synchronous_baseline(cfg, schema, batches)
    assert pipe.final_store_digest == base.final_store_digest
    want, _ = O.pipeline(batches, schema.rows_per_table, schema.emb_dim, cfg.seed, cfg.num_trainers,
                         cfg.cache_capacity, pipe.initial_lookahead, cfg.rpc_batch_proportion)
    table = pipe.final_store.table_view()
    base_idx = schema.table_base()
    for key, row in want.values.items():
        t, r = key >> 44, key & ((1 << 44) - 1)
        np.testing.assert_array_equal(table[base_idx[t] + r, :schema.emb_dim], row)
    assert len(want.values) > 0
    return pipe


def test_avazu_shape():
    schema = Schema(22, AVAZU_ROWS, 1, 16)
    assert 9_000_000 < schema.total_rows < 10_000_000
    rows, labels, dense = generate_columns(ZipfSpec(schema, 1.05, 6 * 4096, seed=3))
    batches = batchify_columns(rows, labels, dense, 4096)
    cfg = _engine().EngineConfig(cache_capacity=schema.total_rows // 100, batch_size=4096, lookahead=4,
                                 num_trainers=2, num_shards=4, seed=11)
    _run_and_compare(schema, batches, cfg)


def test_terabyte_like_shape_dim64():
    """26 tables, D=64 (256-byte rows), cardinalities scaled down 1/100 from
    the Terabyte shape so the pinned store stays small."""
    rows_tb = (3980, 3_980_000, 3_480_000, 2_200_000, 3_000, 1_000, 6_000, 1_000, 1, 40_000, 59_000, 3_800_000,
               300, 20, 14_000, 1_600_000, 10, 5_000, 2_000, 4, 3_300_000, 19, 15, 290_000, 100, 140_000)
    schema = Schema(26, rows_tb, 13, 64)
    rows, labels, dense = generate_columns(ZipfSpec(schema, 1.05, 4 * 8192, seed=9))
    batches = batchify_columns(rows, labels, dense, 8192)
    cfg = _engine().EngineConfig(cache_capacity=schema.total_rows // 100, batch_size=8192, lookahead=0,
                                 num_trainers=1, num_shards=1, seed=5)
    _run_and_compare(schema, batches, cfg)


@pytest.mark.parametrize("window,cache_pct,zipf", [(50, 40.0, 0.8), (200, 30.0, 1.05), (1000, 20.0, 1.2),
                                                   (50, 8.0, 1.2), (50, 5.0, 0.8), (50, 0.1, 1.05)])
def test_sweep_cells(window, cache_pct, zipf):
    """Config 5 cells (reduced): both sides run (one with pressure halving),
    or both fail at the same iteration with the capacity exceeded (iteration
    1 and 0 in the last two cells)."""
    from paper_2202_12429_b200.errors import CacheCapacityError

    schema = Schema(4, (20_000, 5_000, 300, 7), 0, 8)
    rows, labels, dense = generate_columns(ZipfSpec(schema, zipf, 12 * 512, seed=17))
    batches = batchify_columns(rows, labels, dense, 512)
    cap = max(8, int(schema.total_rows * cache_pct / 100))
    cfg = _engine().EngineConfig(cache_capacity=cap, batch_size=512, lookahead=window, num_trainers=1, seed=2)
    try:
        want, _ = O.pipeline(batches, schema.rows_per_table, schema.emb_dim, cfg.seed, 1, cap, window,
                             cfg.rpc_batch_proportion)
        oracle_fail = None
    except RuntimeError as err:
        oracle_fail = int(re.search(r"at (\d+)", str(err)).group(1))
    if oracle_fail is None:
        pipe = _engine().run_pipeline(cfg, schema, batches)
        table = pipe.final_store.table_view()
        base_idx = schema.table_base()
        for key, row in want.values.items():
            t, r = key >> 44, key & ((1 << 44) - 1)
            np.testing.assert_array_equal(table[base_idx[t] + r, :schema.emb_dim], row)
    else:
        with pytest.raises(CacheCapacityError, match=f"iteration {oracle_fail}"):
            _engine().run_pipeline(cfg, schema, batches)
