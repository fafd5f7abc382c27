"""Edge cases of the GPU path against the pinned CPU oracle: ragged last
batches, empty batches, very large packed keys (schema-less registry mode),
single-row tables (every occurrence the same key), batches larger than the
columnar shared-memory sort (generic radix path), and the largest dims of
the EmbeddingBag kernels."""

from __future__ import annotations

import random

import numpy as np
import pytest

from conftest import unpack
from oracle import bagpipe_oracle as O
from paper_2202_12429_b200.traces import (Batch, EmbeddingKey, Example, Schema, ZipfSpec, batchify_columns,
                                          generate_columns)

pytestmark = pytest.mark.gpu


def _engine():
    from paper_2202_12429_b200 import engine

    return engine


def _digest_pair(schema, batches, cfg):
    eng = _engine()
    pipe = eng.run_pipeline(cfg, schema, batches)
    base = eng.run_synchronous_baseline(cfg, schema, batches)
    want = O.baseline(batches, schema.rows_per_table, schema.emb_dim, cfg.seed, cfg.num_trainers).digest()
    return pipe.final_store_digest, base.final_store_digest, want


@pytest.mark.parametrize("n_examples,batch", [(1000, 64), (777, 100), (130, 128)])
def test_ragged_last_batch(n_examples, batch):
    schema = Schema(3, (500, 40, 3), 2, 4)
    rows, labels, dense = generate_columns(ZipfSpec(schema, 1.05, n_examples, seed=5))
    batches = batchify_columns(rows, labels, dense, batch)
    assert batches[-1].num_examples != batch or n_examples % batch == 0
    cfg = _engine().EngineConfig(cache_capacity=2000, batch_size=batch, lookahead=4, num_trainers=2, seed=3)
    got_pipe, got_base, want = _digest_pair(schema, batches, cfg)
    assert got_pipe == got_base == want


def test_single_row_tables_every_occurrence_one_key():
    """Tables with one row: each batch's keys collapse to T uniques with B
    occurrences each (the longest possible sequential chains)."""
    schema = Schema(2, (1, 1), 0, 8)
    rows = np.zeros((4096, 2), dtype=np.int64)
    labels = (np.arange(4096) % 3 == 0).astype(np.uint8)
    batches = batchify_columns(rows, labels, None, 1024)
    cfg = _engine().EngineConfig(cache_capacity=10, batch_size=1024, lookahead=2, num_trainers=3, seed=9)
    got_pipe, got_base, want = _digest_pair(schema, batches, cfg)
    assert got_pipe == got_base == want


def test_batch_larger_than_columnar_sort():
    """20,000 examples per batch > the 16,384 of one per-table smem sort:
    two chunk sorts per column merged by rank."""
    schema = Schema(2, (50_000, 300), 0, 4)
    rows, labels, dense = generate_columns(ZipfSpec(schema, 1.05, 3 * 20_000, seed=8))
    batches = batchify_columns(rows, labels, dense, 20_000)
    cfg = _engine().EngineConfig(cache_capacity=60_000, batch_size=20_000, lookahead=2, num_trainers=1, seed=4)
    got_pipe, got_base, want = _digest_pair(schema, batches, cfg)
    assert got_pipe == got_base == want


def test_huge_packed_keys_plan_stream():
    """Schema-less keys with table ids up to 2^19 and rows up to 2^43 (the
    registry maps them to dense ids): plans equal the oracle's."""
    from paper_2202_12429_b200 import lookahead as lk

    rng = random.Random(77)
    universe = [EmbeddingKey(rng.randrange(1 << 19), rng.randrange(1 << 43)) for _ in range(40)]
    batches = [Batch(i, [Example(j & 1, (), (rng.choice(universe), rng.choice(universe)))
                         for j in range(rng.randint(1, 12))]) for i in range(25)]
    want, _ = O.plan_stream(batches, 4, 10**6)
    got = list(lk.plan_trace(batches, 4, 10**6))
    assert len(got) == len(want)
    for p, (it, pf, uniq, ttl, _, look) in zip(got, want):
        assert p.iteration == it and p.lookahead == look
        assert p.prefetch == [unpack(int(x)) for x in pf]
        assert p.ttl_updates == [(unpack(int(x)), int(t)) for x, t in zip(uniq, ttl)]


def test_empty_prep_is_valid():
    """A batch prep over zero occurrences: zero uniques, no kernels fail."""
    import torch

    from paper_2202_12429_b200.device import DevicePrep

    prep = DevicePrep(np.zeros(0, np.uint64), np.zeros(0, np.uint8), np.asarray([0, 0]), 0)
    assert prep.num_unique == 0
    torch.cuda.synchronize()


@pytest.mark.parametrize("dim", [4, 32, 128])
def test_embedding_bag_dims(dim):
    """Single-key bags at the smallest and largest supported dims: forward
    exact, backward + SGD within fp32 tolerance of np.add.at."""
    import torch

    from paper_2202_12429_b200 import _lib as L
    from paper_2202_12429_b200.device import DevicePrep
    from paper_2202_12429_b200.traces import pack_keys

    rng = np.random.default_rng(dim)
    n_rows, n = 300, 5000
    idx = np.minimum(rng.zipf(1.2, n) - 1, n_rows - 1).astype(np.int64)
    w = rng.standard_normal((n_rows, dim)).astype(np.float32)
    g = rng.standard_normal((n, dim)).astype(np.float32)
    prep = DevicePrep(pack_keys(np.zeros_like(idx), idx), np.zeros(n, np.uint8), np.asarray([0, n]), 0, occ_index=2)
    slots = torch.empty(prep.num_unique, dtype=torch.int32, device="cuda")
    lib = L.lib()
    L.check(lib.bp_prep_key_rows(prep.handle, L.ptr(slots), L.stream_ptr()), "key rows")
    d_w = torch.from_numpy(w).cuda()
    pooled = torch.empty((n, dim), dtype=torch.float32, device="cuda")
    L.check(lib.bp_embbag_forward(prep.handle, L.ptr(d_w), dim, L.ptr(slots), dim, None, n, 0, None, L.ptr(pooled),
                                  L.stream_ptr()), "fwd")
    assert torch.equal(pooled.cpu(), torch.from_numpy(w[idx]))
    d_g = torch.from_numpy(g).cuda()
    L.check(lib.bp_embbag_backward(prep.handle, L.ptr(d_g), None, None, L.ptr(d_w), dim, L.ptr(slots), None, dim, 0,
                                   0.1, 0.0, None, L.stream_ptr()), "bwd")
    gs = np.zeros_like(w)
    np.add.at(gs, idx, g)
    np.testing.assert_allclose(d_w.cpu().numpy(), w - np.float32(0.1) * gs, rtol=1e-5, atol=2e-4)
