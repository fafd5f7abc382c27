"""Trace data model and host plumbing (reference tests/test_traces.py shape);
the columnar generator is pinned to digests recorded from the reference."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden
from paper_2202_12429_b200.errors import ConfigurationError, TraceFormatError
from paper_2202_12429_b200.hashing import fnv1a64, fnv1a64_u64s, splitmix64
from paper_2202_12429_b200.traces import (
    Batch,
    EmbeddingKey,
    Example,
    Schema,
    ZipfSpec,
    batchify,
    batchify_columns,
    generate_columns,
    generate_synthetic_trace,
    hash_categorical,
    iter_trace,
    pack_keys,
    read_trace_columns,
    read_trace_schema,
    unpack_keys,
    write_trace,
    write_trace_columns,
)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", ["small", "mixed", "acceptance"])
def test_columnar_generator_is_the_reference_stream(name):
    g = golden("generator.json")[name]
    nt, rows, nd, dim = g["schema"]
    r, lab, dense = generate_columns(ZipfSpec(Schema(nt, rows, nd, dim), g["exponent"], g["n"], g["seed"]))
    assert (sha(r), sha(lab), sha(dense)) == (g["rows_sha"], g["labels_sha"], g["dense_sha"])


def test_hash_vectors_match_reference():
    g = golden("hashing.json")
    for s, want in g["fnv_bytes"]:
        assert hex(fnv1a64(s.encode())) == want
    for words, want in g["fnv_u64s"]:
        assert fnv1a64_u64s(*words) == want
    for x, want in g["splitmix"]:
        assert splitmix64(x) == want


def test_hash_categorical():
    assert hash_categorical("0", 7) == fnv1a64(bytes(8)) % 7
    assert hash_categorical("68fd1e64", 1) == 0
    with pytest.raises(ConfigurationError):
        hash_categorical("1", 0)


def test_object_and_columnar_batches_agree(small_schema):
    spec = ZipfSpec(small_schema, 1.05, 200, seed=3)
    objs = list(batchify(generate_synthetic_trace(spec), 64))
    rows, labels, dense = generate_columns(spec)
    cols = batchify_columns(rows, labels, dense, 64)
    assert [b.iteration for b in objs] == [b.iteration for b in cols] == [0, 1, 2, 3]
    for a, b in zip(objs, cols):
        ka, la, oa = a.packed_occurrences()
        kb, lb, ob = b.packed_occurrences()
        assert np.array_equal(ka, kb) and np.array_equal(la, lb) and np.array_equal(oa, ob)
        assert a.unique_keys() == b.unique_keys()
        assert a.rank_bounds(3).tolist() == b.rank_bounds(3).tolist()


def test_unique_keys_first_occurrence_order():
    b = Batch(0, [Example(0, (), (EmbeddingKey(0, 3), EmbeddingKey(1, 3))),
                  Example(1, (), (EmbeddingKey(0, 1), EmbeddingKey(1, 3)))])
    assert b.unique_keys() == [EmbeddingKey(0, 3), EmbeddingKey(1, 3), EmbeddingKey(0, 1)]


def test_pack_order_equals_key_order():
    keys = [EmbeddingKey(2, 5), EmbeddingKey(0, 9), EmbeddingKey(1, 0), EmbeddingKey(0, 2)]
    packed = pack_keys([k[0] for k in keys], [k[1] for k in keys])
    assert unpack_keys(np.sort(packed)) == sorted(keys)


def test_batchify_sizes():
    ex = [Example(0, (), (EmbeddingKey(0, i),)) for i in range(5)]
    assert [len(b.examples) for b in batchify(ex, 2)] == [2, 2, 1]
    assert list(batchify([], 4)) == []
    with pytest.raises(ConfigurationError):
        list(batchify(ex, 0))


def test_trace_file_round_trip(tmp_path, small_schema):
    spec = ZipfSpec(small_schema, 1.05, 300, seed=9)
    a, b = str(tmp_path / "a.trace"), str(tmp_path / "b.trace")
    assert write_trace(a, small_schema, generate_synthetic_trace(spec)) == 300
    rows, labels, dense = generate_columns(spec)
    write_trace_columns(b, small_schema, rows, labels, dense)
    assert open(a, "rb").read() == open(b, "rb").read()
    assert read_trace_schema(a) == small_schema
    sc, r2, l2, d2 = read_trace_columns(a)
    assert np.array_equal(r2, rows) and np.array_equal(l2, labels) and np.array_equal(d2, dense)
    back = list(iter_trace(a))
    assert back[7] == list(generate_synthetic_trace(spec))[7]
    bad = tmp_path / "bad.trace"
    bad.write_bytes(b"XXXXXX" + open(a, "rb").read()[6:])
    with pytest.raises(TraceFormatError):
        read_trace_schema(str(bad))


def test_schema_validation():
    with pytest.raises(ConfigurationError):
        Schema(2, (10,), 0, 4)
    with pytest.raises(ConfigurationError):
        Schema(1, (0,), 0, 4)
    assert Schema(2, (3, 4), 0, 4).table_base().tolist() == [0, 3, 7]
