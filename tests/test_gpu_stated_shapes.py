"""BASELINE.json configs 3 and 4 at their stated shapes, bit-exact:

* Avazu Wide&Deep shape: 22 tables summing to 9,449,206 rows, D=16, batch
  16,384, 8 batches, HBM cache 1% of rows, auto lookahead;
* Criteo-Terabyte shape: 26 tables with the Terabyte cardinalities scaled
  to 1/10 (88,277,447 rows, a 22.6 GB pinned fp32 store), D=64, batch
  65,536, 5 batches, cache 1% of rows, L=2 (evictions and write-backs every
  iteration).

Checks: the GPU plan stream equals the oracle's plan by plan (sha of
iteration, lookahead, sorted prefetch, first-occurrence ttl updates --
reference lookahead.py:64-123); the pipelined engine's final store digest
equals the synchronous baseline's (reference engine.py:688-769); every row
the run wrote equals the CPU oracle pipeline's row bit for bit."""

from __future__ import annotations

import gc

import numpy as np
import pytest

from oracle import bagpipe_oracle as O
from paper_2202_12429_b200.traces import Schema, ZipfSpec, batchify_columns, generate_columns

pytestmark = pytest.mark.gpu

AVAZU_ROWS = (7, 7, 4737, 7745, 26, 8552, 559, 36, 2686408, 6729486, 8251, 5, 4, 2626, 8, 9, 435, 4, 68, 172,
              60, 1)
# Criteo Terabyte cardinalities (sum 882,774,559 = P:448 "882.77M"), / 10
TB_FULL = (227605432, 39060, 17295, 7424, 20265, 3, 7122, 1543, 63, 130229467, 3067956, 405282, 10, 2209, 11938,
           155, 4, 976, 14, 292775614, 40790948, 187188510, 590152, 12973, 108, 36)
TB_TENTH = tuple(max(1, r // 10) for r in TB_FULL)


def _plan_shas_gpu(batches, schema, lookahead, cap):
    from paper_2202_12429_b200 import lookahead as lk

    state = lk.new_state(lookahead, cap, schema=schema)
    src = iter(batches)
    shas = []
    while (p := lk.emit_next_plan(state, src)) is not None:
        pf = O.pack([k[0] for k in p.prefetch], [k[1] for k in p.prefetch]) if p.prefetch else []
        uniq = O.pack([k[0] for k, _ in p.ttl_updates], [k[1] for k, _ in p.ttl_updates])
        shas.append(O.plan_sha((p.iteration, pf, uniq, [t for _, t in p.ttl_updates], None, p.lookahead)))
        lk.adapt_on_pressure(state)
    return shas


def _written_rows_equal(table, schema, want):
    keys = np.fromiter(want.values.keys(), dtype=np.uint64, count=len(want.values))
    rows = np.stack(list(want.values.values()))
    t = (keys >> np.uint64(44)).astype(np.int64)
    r = (keys & np.uint64((1 << 44) - 1)).astype(np.int64)
    got = table[schema.table_base()[t] + r, :schema.emb_dim]
    np.testing.assert_array_equal(got, rows)
    return keys.size


def _check(schema, batches, cfg, lookahead_plans):
    from paper_2202_12429_b200 import engine

    cap = cfg.cache_capacity
    want_shas = [O.plan_sha(p) for p in O.plan_stream(batches, lookahead_plans, cap)[0]]
    assert _plan_shas_gpu(batches, schema, lookahead_plans, cap) == want_shas
    pipe = engine.run_pipeline(cfg, schema, batches)
    digest = pipe.final_store_digest
    want, _ = O.pipeline(batches, schema.rows_per_table, schema.emb_dim, cfg.seed, cfg.num_trainers, cap,
                         pipe.initial_lookahead, cfg.rpc_batch_proportion)
    assert _written_rows_equal(pipe.final_store.table_view(), schema, want) > 0
    assert pipe.totals["dirty_evictions"] > 0
    del pipe
    gc.collect()  # one pinned store at a time
    base = engine.run_synchronous_baseline(cfg, schema, batches)
    assert base.final_store_digest == digest


def test_avazu_stated_shape():
    from paper_2202_12429_b200.engine import EngineConfig

    schema = Schema(22, AVAZU_ROWS, 1, 16)
    rows, labels, dense = generate_columns(ZipfSpec(schema, 1.05, 8 * 16384, seed=3))
    batches = batchify_columns(rows, labels, dense, 16384)
    cfg = EngineConfig(cache_capacity=schema.total_rows // 100, batch_size=16384, lookahead=0, num_trainers=1,
                       num_shards=1, seed=11)
    _check(schema, batches, cfg, 4)


def test_terabyte_tenth_scale_dim64_batch65536():
    from paper_2202_12429_b200.engine import EngineConfig

    schema = Schema(26, TB_TENTH, 13, 64)
    assert schema.total_rows == 88_277_447
    rows, labels, dense = generate_columns(ZipfSpec(schema, 1.05, 5 * 65536, seed=9))
    batches = batchify_columns(rows, labels, None, 65536)
    cfg = EngineConfig(cache_capacity=schema.total_rows // 100, batch_size=65536, lookahead=2, num_trainers=1,
                       num_shards=1, seed=5)
    _check(schema, batches, cfg, 2)
