"""GPU cache / store / trainer units against the reference contracts
(reference tests/test_cache.py, tests/test_store.py, tests/test_trainer.py)
and the pinned CPU oracle."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import bagpipe_oracle as O
from paper_2202_12429_b200.errors import (
    CacheCapacityError,
    CacheMissError,
    CacheOrderingError,
    ConfigurationError,
    StoreError,
    StoreKeyError,
)
from paper_2202_12429_b200.traces import EmbeddingKey, Example, Schema

pytestmark = pytest.mark.gpu


def k(row: int, table: int = 0) -> EmbeddingKey:
    return EmbeddingKey(table, row)


def cache(capacity=4, dim=2):
    from paper_2202_12429_b200.cache import DynamicCache

    return DynamicCache(capacity, dim)


def vec(*xs):
    return np.asarray([xs], dtype=np.float32)


# ------------------------------------------------------------------ cache
def test_insert_and_lookup():
    c = cache()
    c.apply_prefetch([k(3)], vec(1.0, 2.0), {k(3): 2})
    assert k(3) in c and len(c) == 1
    assert c.ttl_of(k(3)) == 2 and not c.is_dirty(k(3))
    np.testing.assert_array_equal(c.lookup_batch([k(3)]), [[1.0, 2.0]])


def test_capacity_duplicate_missing_ttl():
    c = cache(capacity=1)
    c.apply_prefetch([k(1)], vec(0, 0), {k(1): 1})
    with pytest.raises(CacheCapacityError):
        c.apply_prefetch([k(2)], vec(0, 0), {k(2): 1})
    c2 = cache()
    c2.apply_prefetch([k(1)], vec(0, 0), {k(1): 1})
    with pytest.raises(CacheOrderingError):
        c2.apply_prefetch([k(1)], vec(0, 0), {k(1): 1})
    with pytest.raises(CacheOrderingError):
        cache().apply_prefetch([k(5)], vec(0, 0), {})


def test_ttl_updates():
    c = cache()
    c.apply_prefetch([k(3)], vec(0, 0), {k(3): 2})
    c.apply_ttl_updates([(k(3), 3)])
    assert c.ttl_of(k(3)) == 3
    with pytest.raises(CacheOrderingError):
        c.apply_ttl_updates([(k(9), 1)])


def test_lookup_order_miss_and_copy():
    c = cache()
    c.apply_prefetch([k(1), k(2)], np.asarray([[1, 1], [2, 2]], np.float32), {k(1): 5, k(2): 5})
    np.testing.assert_array_equal(c.lookup_batch([k(2), k(1)]), [[2, 2], [1, 1]])
    with pytest.raises(CacheMissError) as err:
        c.lookup_batch([k(1), k(7)], iteration=42)
    assert err.value.key == k(7) and err.value.iteration == 42
    assert c.lookup_batch([]).shape == (0, 2)
    out = c.lookup_batch([k(1)])
    out[0, 0] = 99
    np.testing.assert_array_equal(c.lookup_batch([k(1)]), [[1.0, 1.0]])


def test_update_and_eviction_sorted_with_dirty():
    c = cache(capacity=8)
    keys = [k(5), k(2), k(1, table=1)]
    c.apply_prefetch(keys, np.zeros((3, 2), np.float32), {key: 1 for key in keys})
    c.update_rows(c.resolve_slots([k(2)]), vec(3, 4), np.asarray([True]))
    out = c.evict_expired(1)
    assert [key for key, _, _ in out] == [k(2), k(5), k(1, table=1)]
    assert [d for _, _, d in out] == [True, False, False]
    np.testing.assert_array_equal(out[0][1], [3, 4])
    assert len(c) == 0
    with pytest.raises(CacheOrderingError):
        c.evict_expired(0)


def test_checksum_and_digest_sensitivity():
    a, b = cache(), cache()
    for c in (a, b):
        c.apply_prefetch([k(1), k(2)], np.asarray([[1, 2], [3, 4]], np.float32), {k(1): 3, k(2): 4})
    assert a.content_checksum() == b.content_checksum()
    assert a.canonical_digest() == b.canonical_digest()
    b.write_local_update(k(1), np.asarray([1, 2.0000002], np.float32))
    assert a.content_checksum() != b.content_checksum()
    assert a.canonical_digest() != b.canonical_digest()


def test_slot_reuse_and_growth():
    c = cache(capacity=600, dim=2)
    keys = [k(i) for i in range(600)]
    c.apply_prefetch(keys, np.zeros((600, 2), np.float32), {key: 1 for key in keys})
    assert len(c) == 600 and c.peak_occupancy == 600 and c.insertions == 600
    c.evict_expired(1)
    assert c.evictions == 600 and len(c) == 0
    c.apply_prefetch(keys[:10], np.ones((10, 2), np.float32), {key: 2 for key in keys[:10]})
    assert len(c) == 10
    with pytest.raises(ConfigurationError):
        cache(capacity=0)


# ------------------------------------------------------------------ store
SCHEMA = Schema(2, (100, 50), 0, 4)


def store(seed=0, shards=2, schema=SCHEMA):
    from paper_2202_12429_b200.store import ShardedStore

    return ShardedStore(schema, shards, seed)


def test_initial_values_match_reference_golden():
    from paper_2202_12429_b200.store import initial_values

    for seed, tables, rows, bits in golden("hashing.json")["init"]:
        got = initial_values(Schema(3, (7, 50000, 3), 0, 16), seed, tables, rows)
        assert got.view(np.uint32).tolist() == bits


def test_store_fetch_write_digest():
    s = store(seed=1)
    vals = s.fetch([k(r) for r in range(100)])
    assert (vals >= -0.05).all() and (vals < 0.05).all()
    np.testing.assert_array_equal(vals, O.init_rows(1, [0] * 100, range(100), 4))
    assert s.snapshot_digest() == store(seed=1, shards=4).snapshot_digest()
    assert s.snapshot_digest() != store(seed=2).snapshot_digest()
    s.write_back([k(3), k(1, table=1)], np.ones((2, 4), np.float32))
    np.testing.assert_array_equal(s.fetch([k(3)]), np.ones((1, 4)))
    assert [key for key, _ in s.written_items()] == [k(3), k(1, table=1)]
    with pytest.raises(StoreKeyError):
        s.fetch([k(100)])
    with pytest.raises(StoreKeyError):
        s.fetch([k(0, table=2)])
    with pytest.raises(StoreError):
        s.write_back([k(1), k(1)], np.zeros((2, 4), np.float32))
    before = s.snapshot_digest()
    v = s.fetch([k(7)])
    v[0, 0] = np.nextafter(v[0, 0], np.float32(1))
    s.write_back([k(7)], v)
    assert s.snapshot_digest() != before


def test_store_lazy_fetch_equals_host_gather():
    """bp_store_fetch_lazy (init computed on the GPU for never-written rows)
    returns exactly what the full host-table gather returns."""
    import torch

    from paper_2202_12429_b200 import _lib as L
    from paper_2202_12429_b200.traces import pack_keys

    s = store(seed=5)
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(100, 60, replace=False))
    s.write_back([k(int(r)) for r in rows[::3]], rng.standard_normal((len(rows[::3]), 4)).astype(np.float32))
    ids = torch.from_numpy(rows.astype(np.uint32)).cuda()
    keys = torch.from_numpy(pack_keys(np.zeros_like(rows), rows)).cuda()
    lazy = s.fetch_ids_async(ids, len(rows), d_keys=keys)
    full = s.fetch_ids_async(ids, len(rows))
    torch.cuda.synchronize()
    assert torch.equal(lazy, full)
    assert L.lib() is not None


def test_store_dump_round_trip(tmp_path):
    from paper_2202_12429_b200.store import read_store_dump, write_store_dump

    s = store(seed=3)
    s.write_back([k(5), k(2, table=1)], np.arange(8, dtype=np.float32).reshape(2, 4))
    path = str(tmp_path / "d.store")
    assert write_store_dump(s, path) == 2
    assert read_store_dump(path).snapshot_digest() == s.snapshot_digest()


# ---------------------------------------------------------------- trainer
def test_gradient_core_matches_scalar_oracle():
    from paper_2202_12429_b200.trainer import StubModelConfig, gradient_core

    rng = np.random.default_rng(0)
    cfg = StubModelConfig()
    for _ in range(20):
        u = int(rng.integers(1, 30))
        n = int(rng.integers(1, 200))
        idx = rng.integers(0, u, size=n)
        labels = rng.integers(0, 2, size=n).astype(np.float32)
        vals = rng.standard_normal((u, 5)).astype(np.float32)
        scaled = np.float32(cfg.c_value) * vals
        occ = scaled[idx] + (np.float32(cfg.c_label) * (labels - np.float32(0.5)))[:, None]
        want = np.zeros_like(vals)
        np.add.at(want, idx, occ)
        np.testing.assert_array_equal(gradient_core(idx, labels, vals, cfg), want)


def test_combine_rank_order_and_sgd():
    from paper_2202_12429_b200.trainer import combine_core, sgd_step

    rng = np.random.default_rng(1)
    blocks = [rng.standard_normal((4, 3)).astype(np.float32) * np.float32(10.0) ** int(rng.integers(-4, 4)) for _ in range(3)]
    idx = [np.asarray([0, 1, 2, 3]), np.asarray([2, 0, 1, 3]), np.asarray([3, 2, 1, 0])]
    want = np.zeros((4, 3), np.float32)
    np.add.at(want, np.concatenate(idx), np.concatenate(blocks))
    np.testing.assert_array_equal(combine_core(idx, blocks, 4, 3), want)
    v = rng.standard_normal((7, 3)).astype(np.float32)
    g = rng.standard_normal((7, 3)).astype(np.float32)
    np.testing.assert_array_equal(sgd_step(v, g, 0.01), v - np.float32(0.01) * g)


def test_label_only_term_and_local_gradients():
    from paper_2202_12429_b200.trainer import StubModelConfig, local_gradients

    cfg = StubModelConfig(c_value=0.0)
    grads = local_gradients([Example(1, (), (k(1),))], {k(1): np.ones(4, np.float32)}, cfg)
    np.testing.assert_array_equal(grads[k(1)], np.full(4, np.float32(0.0005)))
    with pytest.raises(CacheMissError):
        local_gradients([Example(1, (), (k(2),))], {}, cfg)


# ---------------------------------------------------------------- prep
@pytest.mark.parametrize("batch", [16384, 40000])
def test_columnar_prep_equals_generic_prep(batch):
    """The per-column shared-memory sort (for > 16,384 examples: chunk sorts
    merged by rank) and the generic global radix sort produce identical
    preps (order of every array), incl. trainer ranks."""
    import ctypes as C

    import torch

    from paper_2202_12429_b200 import _lib as L
    from paper_2202_12429_b200.device import DevicePrep
    from paper_2202_12429_b200.traces import ZipfSpec, batchify_columns, generate_columns

    schema = Schema(5, (3, 70_000, 1000, 5_000_000, 17), 0, 4)
    rows, labels, _ = generate_columns(ZipfSpec(schema, 1.1, 2 * batch, seed=9))
    for b in batchify_columns(rows, labels, None, batch):
        keys, labs, _ = b.packed_occurrences()
        rb = b.rank_bounds(3)
        col = DevicePrep(keys, labs, rb, b.iteration, schema, columns=(b.num_examples, b.table_ids()))
        gen = DevicePrep(keys, labs, rb, b.iteration, schema)
        u = gen.num_unique
        assert col.num_unique == u
        n = gen.n_occ
        for name, dt, cnt in (("d_uniq_key_s", torch.uint64, u), ("d_uniq_id_s", torch.uint32, u),
                              ("d_uniq_key_k", torch.uint64, u), ("d_perm_s2k", torch.uint32, u),
                              ("d_seg_start", torch.uint32, u + 1), ("d_occ_pos", torch.uint32, n),
                              ("d_occ_label", torch.uint8, n)):
            assert torch.equal(col.tensor(name, dt, cnt).cpu(), gen.tensor(name, dt, cnt).cpu()), name
