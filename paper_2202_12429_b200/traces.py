"""Trace data model: keys, schemas, examples and (columnar) batches.

API-compatible with the reference data model (reference ``traces.py:35-103``)
but stored column-wise: a :class:`Batch` built by :func:`batchify_columns` or
:func:`read_trace_columns` holds ``rows[n, num_tables]`` and ``labels[n]``
numpy arrays and never materialises Python ``Example`` objects unless a caller
asks for ``.examples``.  The hot path only ever sees
:meth:`Batch.packed_occurrences` -- the u64 keys ``(table << 44) | row`` in
occurrence order (reference ``engine.py:117-121``) -- which are uploaded to
HBM and deduplicated there by the CUDA batch-prep kernels.

The synthetic generator replays the reference generator's numpy stream
column by column (reference ``traces.py:175-209``): per table
``rng.permutation(rows)`` then ``rng.choice(rows, n, p=rank^-s)``; labels
``(i + seed) & 1``; dense features ``unit(splitmix64(seed ^ fnv(i, col)))``.
``tests/test_traces.py`` pins it to digests recorded from the reference.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass
from typing import BinaryIO, Iterable, Iterator, NamedTuple

import numpy as np

from .errors import ConfigurationError, RecordParseError, SchemaError, TraceFormatError
from .hashing import fnv1a64_u64_arrays, fnv1a64_u64s, splitmix64_array, unit_from_u64_array

TRACE_MAGIC = b"EMTRC1"
TRACE_VERSION = 1
KEY_TABLE_SHIFT = 44  # packed key = (table << 44) | row; row < 2**44


class EmbeddingKey(NamedTuple):
    """One row of one table; ordering is (table_id, row_id) lexicographic."""

    table_id: int
    row_id: int


@dataclass(frozen=True)
class Schema:
    """Embedding-table shapes plus the dense-feature count (reference traces.py:42-71)."""

    num_tables: int
    rows_per_table: tuple
    num_dense: int
    emb_dim: int

    def __post_init__(self):
        object.__setattr__(self, "rows_per_table", tuple(int(r) for r in self.rows_per_table))
        if self.num_tables < 1:
            raise ConfigurationError("num_tables must be >= 1")
        if len(self.rows_per_table) != self.num_tables:
            raise ConfigurationError(
                f"rows_per_table has {len(self.rows_per_table)} entries, expected {self.num_tables}"
            )
        if any(r < 1 for r in self.rows_per_table):
            raise ConfigurationError("every table needs at least one row")
        if self.num_dense < 0:
            raise ConfigurationError("num_dense must be >= 0")
        if self.emb_dim < 1:
            raise ConfigurationError("emb_dim must be >= 1")

    @property
    def total_rows(self) -> int:
        return sum(self.rows_per_table)

    def contains_key(self, key: EmbeddingKey) -> bool:
        return 0 <= key.table_id < self.num_tables and 0 <= key.row_id < self.rows_per_table[key.table_id]

    def table_base(self) -> np.ndarray:
        """Global row index of each table's row 0: ``g = base[t] + row`` is
        monotone in (table, row), so it doubles as the HBM row index and as
        an order-preserving 32-bit sort key."""
        base = np.zeros(self.num_tables + 1, dtype=np.int64)
        np.cumsum(np.asarray(self.rows_per_table, dtype=np.int64), out=base[1:])
        return base


@dataclass(slots=True)
class Example:
    """Click label, dense features and one key per table."""

    label: int
    dense: tuple
    sparse: tuple


def pack_keys(tables, rows) -> np.ndarray:
    """Packed u64 keys ``(table << 44) | row``; numeric order == key order."""
    t = np.asarray(tables, dtype=np.uint64)
    r = np.asarray(rows, dtype=np.uint64)
    return (t << np.uint64(KEY_TABLE_SHIFT)) | r


def unpack_key(packed: int) -> EmbeddingKey:
    packed = int(packed)
    return EmbeddingKey(packed >> KEY_TABLE_SHIFT, packed & ((1 << KEY_TABLE_SHIFT) - 1))


def unpack_keys(packed) -> list:
    arr = np.asarray(packed, dtype=np.uint64)
    t = (arr >> np.uint64(KEY_TABLE_SHIFT)).tolist()
    r = (arr & np.uint64((1 << KEY_TABLE_SHIFT) - 1)).tolist()
    return [EmbeddingKey(a, b) for a, b in zip(t, r)]


class Batch:
    """A numbered group of consecutive examples (reference traces.py:83-103).

    Either object-backed (``Batch(iteration, examples)``, the reference's
    constructor) or column-backed (:meth:`from_columns`).  ``_memo`` caches
    derived host arrays and device-side batch preps, like the reference's
    memo dict.
    """

    __slots__ = ("iteration", "_examples", "rows", "labels", "dense", "tables", "_memo", "_n_ex")

    def __init__(self, iteration: int, examples=None, *, rows=None, labels=None, dense=None, tables=None):
        self.iteration = int(iteration)
        self._examples = examples
        self.rows = rows
        self.labels = labels
        self.dense = dense
        # table id of each column (default: column index); a table-wise shard
        # keeps the global ids of its tables (shard.py)
        self.tables = None if tables is None else np.asarray(tables, dtype=np.int64)
        self._memo: dict = {}
        self._n_ex = None
        if examples is None and rows is None:
            self._examples = []

    @classmethod
    def from_columns(cls, iteration: int, rows: np.ndarray, labels: np.ndarray, dense=None, tables=None) -> "Batch":
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        if rows.ndim != 2:
            raise ConfigurationError("rows must be [examples, tables]")
        labels = np.ascontiguousarray(labels, dtype=np.uint8)
        if labels.shape != (rows.shape[0],):
            raise ConfigurationError("labels must be [examples]")
        if tables is not None and len(tables) != rows.shape[1]:
            raise ConfigurationError("one table id per column")
        return cls(iteration, None, rows=rows, labels=labels, dense=dense, tables=tables)

    @classmethod
    def from_occurrences(cls, iteration: int, keys: np.ndarray, labels: np.ndarray, offsets: np.ndarray) -> "Batch":
        """Occurrence-backed batch: packed keys u64[n_occ] in occurrence order,
        one label byte per occurrence and the example offsets i64[n+1] -- the
        layout of a row-wise shard (shard.row_shard_batches), whose examples
        carry a variable number of the rank's keys.  Examples are built only
        when read."""
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        labels = np.ascontiguousarray(labels, dtype=np.uint8)
        if offsets.ndim != 1 or offsets.size < 1 or offsets[0] != 0 or offsets[-1] != keys.size:
            raise ConfigurationError("offsets must run from 0 to the occurrence count")
        if labels.shape != keys.shape:
            raise ConfigurationError("one label per occurrence")
        b = cls(iteration, None, rows=None)
        b._examples = None
        b._n_ex = offsets.size - 1
        b._memo["occ"] = (keys, labels, offsets)
        return b

    def table_ids(self) -> np.ndarray:
        return self.tables if self.tables is not None else np.arange(self.rows.shape[1], dtype=np.int64)

    @property
    def is_columnar(self) -> bool:
        return self._examples is None and self._n_ex is None

    @property
    def examples(self) -> list:
        if self._examples is None and self._n_ex is not None:  # occurrence-backed
            keys, labels, offsets = self._memo["occ"]
            ks = unpack_keys(keys)
            self._examples = [Example(int(labels[offsets[i]]) if offsets[i + 1] > offsets[i] else 0, (),
                                      tuple(ks[offsets[i]:offsets[i + 1]])) for i in range(self._n_ex)]
        if self._examples is None:
            n, nt = self.rows.shape
            dense = self.dense
            out = []
            tids = self.table_ids().tolist()
            for i in range(n):
                d = tuple(float(v) for v in dense[i]) if dense is not None else ()
                out.append(Example(int(self.labels[i]), d,
                                   tuple(EmbeddingKey(tids[c], int(self.rows[i, c])) for c in range(nt))))
            self._examples = out
        return self._examples

    @property
    def num_examples(self) -> int:
        if self._n_ex is not None:
            return self._n_ex
        return self.rows.shape[0] if self._examples is None else len(self._examples)

    def __len__(self) -> int:
        return self.num_examples

    def __repr__(self) -> str:
        return f"Batch(iteration={self.iteration}, examples={self.num_examples})"

    def pin_memory(self) -> "Batch":
        """Keep the batch in pinned host memory, so the engine DMAs it straight
        to the GPU (no staging copy): a columnar batch whose row ids fit in 32
        bits as its row ids, each column at 1, 2 or 4 bytes, + per-example
        labels (the compact upload), any other batch as its packed
        occurrences (keys, labels)."""
        import torch

        if self._examples is None and self.rows is not None and self.rows.size and \
                0 <= int(self.rows.min()) and int(self.rows.max()) < (1 << 32):
            # each column at the narrowest width its row ids fit (u32 / u16 /
            # u8), the planes in that order in one pinned buffer
            mx = self.rows.max(axis=0)
            widths = np.where(mx < (1 << 8), 1, np.where(mx < (1 << 16), 2, 4)).astype(np.int8)
            n = self.rows.shape[0]
            planes = [np.ascontiguousarray(self.rows[:, widths == w], dtype=dt)
                      for w, dt in ((4, np.uint32), (2, np.uint16), (1, np.uint8))]
            nbytes = sum(p.nbytes for p in planes)
            buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
            off = 0
            for p in planes:
                buf.numpy()[off:off + p.nbytes] = p.reshape(-1).view(np.uint8)
                off += p.nbytes
            pl = torch.empty(n, dtype=torch.uint8, pin_memory=True)
            pl.numpy()[:] = self.labels
            self._memo["pinned_planes"] = (buf, pl, widths)
            return self
        keys, labels, offsets = self.packed_occurrences()
        pk = torch.empty(keys.size, dtype=torch.uint64, pin_memory=True)
        pl = torch.empty(labels.size, dtype=torch.uint8, pin_memory=True)
        pk.numpy()[:] = keys
        pl.numpy()[:] = labels
        self._memo["pinned"] = (pk, pl)  # owners of the pinned memory
        self._memo["occ"] = (pk.numpy(), pl.numpy(), offsets)
        return self

    def packed_occurrences(self) -> tuple:
        """(keys u64[n_occ], labels u8[n_occ], example_offsets i64[n+1]).

        Occurrence order is examples in order, keys of an example in order --
        the order every reference accumulation follows (trainer.py:48-53).
        """
        memo = self._memo.get("occ")
        if memo is not None:
            return memo
        if self._examples is None:
            n, nt = self.rows.shape
            keys = pack_keys(self.table_ids().astype(np.uint64)[None, :], self.rows).reshape(-1)
            labels = np.repeat(self.labels, nt)
            offsets = np.arange(n + 1, dtype=np.int64) * nt
        else:
            tables, rows, labels, counts = [], [], [], []
            for ex in self._examples:
                counts.append(len(ex.sparse))
                for key in ex.sparse:
                    tables.append(key[0])
                    rows.append(key[1])
                    labels.append(ex.label)
            keys = pack_keys(np.asarray(tables, dtype=np.int64), np.asarray(rows, dtype=np.int64))
            labels = np.asarray(labels, dtype=np.uint8)
            offsets = np.zeros(len(counts) + 1, dtype=np.int64)
            np.cumsum(np.asarray(counts, dtype=np.int64), out=offsets[1:])
        memo = (np.ascontiguousarray(keys, dtype=np.uint64), labels, offsets)
        self._memo["occ"] = memo
        return memo

    def rank_bounds(self, num_trainers: int) -> np.ndarray:
        """Occurrence-position bounds of the T contiguous trainer sub-batches:
        rank r owns examples ``[r*n//T, (r+1)*n//T)`` (reference engine.py:159-161)."""
        _, _, offsets = self.packed_occurrences()
        n = len(offsets) - 1
        ex = [(r * n) // num_trainers for r in range(num_trainers + 1)]
        return offsets[np.asarray(ex, dtype=np.int64)].astype(np.int64)

    def unique_keys(self) -> list:
        """Unique keys in first-occurrence order (reference traces.py:91-103).

        Host convenience for API callers; the planner and engine dedupe on
        the device (``csrc/prep.cu``) and never call this.
        """
        cached = self._memo.get("unique")
        if cached is None:
            keys, _, _ = self.packed_occurrences()
            if len(keys) == 0:
                cached = []
            else:
                _, first = np.unique(keys, return_index=True)
                cached = unpack_keys(keys[np.sort(first)])
            self._memo["unique"] = cached
        return cached


@dataclass(frozen=True)
class ZipfSpec:
    """Synthetic skewed workload parameters (reference traces.py:106-119)."""

    schema: Schema
    exponent: float
    num_examples: int
    seed: int

    def __post_init__(self):
        if not self.exponent > 0:
            raise ConfigurationError("zipf exponent must be > 0")
        if self.num_examples < 0:
            raise ConfigurationError("num_examples must be >= 0")


def hash_categorical(token: str, table_rows: int) -> int:
    """Hex token -> row: FNV-1a 64 of its low 64 bits mod table size."""
    if table_rows < 1:
        raise ConfigurationError("table_rows must be >= 1")
    try:
        raw = int(token, 16)
    except ValueError:
        raise RecordParseError(f"not a hexadecimal token: {token!r}") from None
    return fnv1a64_u64s(raw) % table_rows


def parse_criteo_tsv(path: str, schema: Schema) -> Iterator[Example]:
    """Criteo TSV -> Examples (label, log1p dense rounded to f32, hashed keys)."""
    expected = 1 + schema.num_dense + schema.num_tables
    with open(path, "r", encoding="ascii") as fh:
        for lineno, line in enumerate(fh, start=1):
            cols = line.rstrip("\n").split("\t")
            if len(cols) != expected:
                raise SchemaError(f"line {lineno}: expected {expected} columns, got {len(cols)}")
            try:
                label = int(cols[0])
                if label not in (0, 1):
                    raise RecordParseError(f"label must be 0 or 1, got {cols[0]!r}")
                dense = tuple(
                    0.0 if c == "" else float(np.float32(math.log1p(int(c))))
                    for c in cols[1 : 1 + schema.num_dense]
                )
                sparse = tuple(
                    EmbeddingKey(t, 0 if c == "" else hash_categorical(c, schema.rows_per_table[t]))
                    for t, c in enumerate(cols[1 + schema.num_dense :])
                )
            except RecordParseError as exc:
                raise RecordParseError(str(exc), line=lineno) from None
            except ValueError as exc:
                raise RecordParseError(str(exc), line=lineno) from None
            yield Example(label, dense, sparse)


def generate_columns(spec: ZipfSpec) -> tuple:
    """Columnar synthetic trace: (rows i64[n, T], labels u8[n], dense f32[n, num_dense]).

    Bit-identical to the reference object generator for the same spec: the
    same Generator calls in the same order (permutation then choice per
    table), so the numpy stream is consumed identically.
    """
    schema = spec.schema
    n = spec.num_examples
    rng = np.random.default_rng(spec.seed)
    rows = np.empty((n, schema.num_tables), dtype=np.int64)
    for t, size in enumerate(schema.rows_per_table):
        weights = np.arange(1, size + 1, dtype=np.float64) ** -spec.exponent
        weights /= weights.sum()
        perm = rng.permutation(size)
        rows[:, t] = perm[rng.choice(size, size=n, p=weights)]
    labels = ((np.arange(n, dtype=np.int64) + (spec.seed & 1)) & 1).astype(np.uint8)
    if schema.num_dense:
        ex = np.repeat(np.arange(n, dtype=np.uint64), schema.num_dense)
        col = np.tile(np.arange(schema.num_dense, dtype=np.uint64), n)
        mixed = splitmix64_array(np.uint64(spec.seed & 0xFFFFFFFFFFFFFFFF) ^ fnv1a64_u64_arrays(ex, col))
        dense = unit_from_u64_array(mixed).astype(np.float32).reshape(n, schema.num_dense)
    else:
        dense = np.zeros((n, 0), dtype=np.float32)
    return rows, labels, dense


def generate_synthetic_trace(spec: ZipfSpec) -> Iterator[Example]:
    """Object-stream form of :func:`generate_columns` (reference API)."""
    rows, labels, dense = generate_columns(spec)
    nt = spec.schema.num_tables
    for i in range(spec.num_examples):
        yield Example(
            int(labels[i]),
            tuple(float(v) for v in dense[i]),
            tuple(EmbeddingKey(t, int(rows[i, t])) for t in range(nt)),
        )


def batchify(stream: Iterable[Example], batch_size: int) -> Iterator[Batch]:
    """Group consecutive Examples into batches 0, 1, 2, ...; last may be short."""
    if batch_size < 1:
        raise ConfigurationError("batch_size must be >= 1")
    iteration = 0
    pending: list = []
    for ex in stream:
        pending.append(ex)
        if len(pending) == batch_size:
            yield Batch(iteration, pending)
            iteration += 1
            pending = []
    if pending:
        yield Batch(iteration, pending)


def batchify_columns(rows: np.ndarray, labels: np.ndarray, dense, batch_size: int, base: int = 0) -> list:
    """Columnar batchify: views into the trace arrays, no per-example objects."""
    if batch_size < 1:
        raise ConfigurationError("batch_size must be >= 1")
    n = rows.shape[0]
    out = []
    for i, lo in enumerate(range(0, n, batch_size)):
        hi = min(n, lo + batch_size)
        out.append(
            Batch.from_columns(base + i, rows[lo:hi], labels[lo:hi], None if dense is None else dense[lo:hi])
        )
    return out


def synthetic_batches(spec: ZipfSpec, batch_size: int) -> list:
    rows, labels, dense = generate_columns(spec)
    return batchify_columns(rows, labels, dense, batch_size)


# -- canonical binary trace (reference traces.py:231-296; README "EMTRC1") ----


def _record_dtype(schema: Schema) -> np.dtype:
    fields = [("label", "u1")]
    fields += [(f"d{i}", "<f4") for i in range(schema.num_dense)]
    fields += [(f"t{i}", "<u8") for i in range(schema.num_tables)]
    return np.dtype(fields)  # packed (no alignment), like struct "<B{d}f{t}Q"


def _write_header(fh: BinaryIO, schema: Schema, count: int) -> None:
    fh.write(TRACE_MAGIC)
    fh.write(struct.pack("<BB", TRACE_VERSION, 0))
    fh.write(struct.pack("<III", schema.num_tables, schema.num_dense, schema.emb_dim))
    fh.write(struct.pack(f"<{schema.num_tables}Q", *schema.rows_per_table))
    fh.write(struct.pack("<Q", count))


def _read_header(fh: BinaryIO) -> tuple:
    magic = fh.read(len(TRACE_MAGIC))
    if magic != TRACE_MAGIC:
        raise TraceFormatError(f"bad magic {magic!r}")
    version, _ = struct.unpack("<BB", fh.read(2))
    if version != TRACE_VERSION:
        raise TraceFormatError(f"unsupported trace version {version}")
    num_tables, num_dense, emb_dim = struct.unpack("<III", fh.read(12))
    rows = struct.unpack(f"<{num_tables}Q", fh.read(8 * num_tables))
    (count,) = struct.unpack("<Q", fh.read(8))
    return Schema(num_tables, rows, num_dense, emb_dim), count


def write_trace(path: str, schema: Schema, examples: Iterable[Example]) -> int:
    """Write the canonical binary trace; returns the example count."""
    rec = struct.Struct(f"<B{schema.num_dense}f{schema.num_tables}Q")
    count = 0
    with open(path, "wb") as fh:
        _write_header(fh, schema, 0)
        count_pos = fh.tell() - 8
        for ex in examples:
            if len(ex.sparse) != schema.num_tables:
                raise SchemaError(f"example {count}: {len(ex.sparse)} keys, schema has {schema.num_tables} tables")
            fh.write(rec.pack(ex.label, *ex.dense, *(k.row_id for k in ex.sparse)))
            count += 1
        fh.seek(count_pos)
        fh.write(struct.pack("<Q", count))
    return count


def write_trace_columns(path: str, schema: Schema, rows, labels, dense) -> int:
    """Columnar writer producing the same bytes as :func:`write_trace`."""
    n = rows.shape[0]
    rec = np.zeros(n, dtype=_record_dtype(schema))
    rec["label"] = labels
    for i in range(schema.num_dense):
        rec[f"d{i}"] = dense[:, i]
    for t in range(schema.num_tables):
        rec[f"t{t}"] = rows[:, t]
    with open(path, "wb") as fh:
        _write_header(fh, schema, n)
        fh.write(rec.tobytes())
    return n


def read_trace_schema(path: str) -> Schema:
    with open(path, "rb") as fh:
        schema, _ = _read_header(fh)
    return schema


def read_trace_columns(path: str) -> tuple:
    """Memory-map an EMTRC1 trace into (schema, rows, labels, dense) columns."""
    with open(path, "rb") as fh:
        schema, count = _read_header(fh)
        offset = fh.tell()
    dt = _record_dtype(schema)
    rec = np.memmap(path, dtype=dt, mode="r", offset=offset, shape=(count,)) if count else np.zeros(0, dt)
    if count and rec.shape[0] != count:
        raise TraceFormatError("truncated trace")
    rows = np.empty((count, schema.num_tables), dtype=np.int64)
    for t in range(schema.num_tables):
        rows[:, t] = rec[f"t{t}"]
    labels = np.ascontiguousarray(rec["label"], dtype=np.uint8)
    dense = np.empty((count, schema.num_dense), dtype=np.float32)
    for i in range(schema.num_dense):
        dense[:, i] = rec[f"d{i}"]
    return schema, rows, labels, dense


def iter_trace(path: str) -> Iterator[Example]:
    """Stream Examples from a canonical trace file."""
    with open(path, "rb") as fh:
        schema, count = _read_header(fh)
        rec = struct.Struct(f"<B{schema.num_dense}f{schema.num_tables}Q")
        for i in range(count):
            buf = fh.read(rec.size)
            if len(buf) != rec.size:
                raise TraceFormatError(f"truncated record {i}")
            fields = rec.unpack(buf)
            rows = fields[1 + schema.num_dense :]
            yield Example(
                fields[0],
                tuple(float(v) for v in fields[1 : 1 + schema.num_dense]),
                tuple(EmbeddingKey(t, rows[t]) for t in range(schema.num_tables)),
            )
