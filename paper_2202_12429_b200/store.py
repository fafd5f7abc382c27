"""Embedding Server on pinned host memory, served by CUDA kernels.

API of reference store.py:65-242 (``ShardedStore``, ``initial_values``, store
dumps).  The whole table is one pinned, GPU-mapped float32 matrix in (table,
row, component) order, created by ``bp_store_create`` (GPU functional init,
reference store.py:29-42); fetch/write-back are zero-copy gather/scatter
kernels over the host link (``bp_store_fetch`` / ``bp_store_write``).  Hash
sharding is kept as placement metadata (``shard_of``): it never changes
values (reference tests/test_store.py:42-45).

The digest is blake2b-128 over the table bytes, i.e. exactly the stream of
reference store.py:179-185, hashed straight from pinned memory.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import struct
import threading

import numpy as np
import torch

from . import _lib as L
from .device import DeviceSchema
from .errors import ConfigurationError, StoreError, StoreKeyError, TraceFormatError
from .hashing import fnv1a64_u64_arrays
from .traces import EmbeddingKey, Schema, pack_keys

DUMP_MAGIC = b"EMSTD1"


def initial_values(schema: Schema, seed: int, tables, rows) -> np.ndarray:
    """Deterministic initial vectors (n, emb_dim), computed on the GPU."""
    t = np.asarray(tables, dtype=np.uint64)
    r = np.asarray(rows, dtype=np.uint64)
    n = len(t)
    if n == 0:
        return np.zeros((0, schema.emb_dim), dtype=np.float32)
    keys = L.to_device((t << np.uint64(44)) | r)
    out = torch.empty((n, schema.emb_dim), dtype=torch.float32, device="cuda")
    L.check(L.lib().bp_init_values(seed & 0xFFFFFFFFFFFFFFFF, schema.emb_dim, L.ptr(keys), n, L.ptr(out),
                                   L.stream_ptr()), "bp_init_values")
    return out.cpu().numpy()


def shard_of_keys(tables, rows, num_shards: int) -> np.ndarray:
    """Shard index of every (table, row): fnv1a64(t, r) mod num_shards
    (reference store.py:80-88, 100-104).  Placement only -- it never changes
    a value -- so it stays host arithmetic."""
    h = fnv1a64_u64_arrays(np.asarray(tables, dtype=np.uint64), np.asarray(rows, dtype=np.uint64))
    return (h % np.uint64(num_shards)).astype(np.int64)


class ShardedStore:
    """All tables behind fetch / write-back; values in pinned host memory."""

    def __init__(self, schema: Schema, num_shards: int, seed: int, _handle=None, _owner=None):
        if num_shards < 1:
            raise ConfigurationError("num_shards must be >= 1")
        self.schema = schema
        self.num_shards = num_shards
        self.seed = seed
        self.dschema = DeviceSchema.get(schema)
        self._lock = threading.Lock()
        self.fetch_calls = 0
        self.write_calls = 0
        self.entries_written = 0
        self._owner = _owner  # native engine owning the store (None: we own it)
        if _handle is None:
            h = C.c_void_p()
            L.check(L.lib().bp_store_create(L.Context.get().handle, self.dschema.handle,
                                            seed & 0xFFFFFFFFFFFFFFFF, L.stream_ptr(), C.byref(h)),
                    "bp_store_create")
        else:
            h = C.c_void_p(_handle)
        self.handle = h
        addr = L.lib().bp_store_host_table(h)
        count = schema.total_rows * schema.emb_dim
        self._table = np.ctypeslib.as_array((C.c_float * count).from_address(addr)).reshape(
            schema.total_rows, schema.emb_dim)
        self._base = schema.table_base()

    def __del__(self):
        try:
            if getattr(self, "handle", None) and getattr(self, "_owner", None) is None:
                torch.cuda.synchronize()
                L.lib().bp_store_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    # -- placement -----------------------------------------------------------
    def shard_of(self, key: EmbeddingKey) -> int:
        return int(shard_of_keys([key[0]], [key[1]], self.num_shards)[0])

    # -- key validation (reference store.py:90-98) ---------------------------
    def _ids(self, keys) -> np.ndarray:
        arr = np.asarray(keys, dtype=np.int64).reshape(len(keys), 2)
        tables, rows = arr[:, 0], arr[:, 1]
        if (tables < 0).any() or (tables >= self.schema.num_tables).any():
            raise StoreKeyError("table id outside schema")
        limits = np.asarray(self.schema.rows_per_table, dtype=np.int64)[tables]
        if (rows < 0).any() or (rows >= limits).any():
            raise StoreKeyError("row id outside table")
        return (self._base[tables] + rows).astype(np.uint32)

    # -- device-path entry points used by the engine -------------------------
    def fetch_ids_async(self, d_ids: torch.Tensor, n: int, d_n=None, stream=None, d_keys=None) -> torch.Tensor:
        """Gather rows for dense ids already on the device (no host round trip).
        With the packed keys (d_keys), never-written rows are computed on the
        GPU (functional init) instead of read over the host link."""
        out = torch.empty((max(n, 0), self.schema.emb_dim), dtype=torch.float32, device="cuda")
        if n > 0:
            if d_keys is not None:
                L.check(L.lib().bp_store_fetch_lazy(self.handle, L.ptr(d_ids), L.ptr(d_keys), n, L.ptr(d_n),
                                                    L.ptr(out), L.stream_ptr(stream)), "bp_store_fetch_lazy")
            else:
                L.check(L.lib().bp_store_fetch(self.handle, L.ptr(d_ids), n, L.ptr(d_n), L.ptr(out),
                                               L.stream_ptr(stream)), "bp_store_fetch")
        return out

    def write_ids_async(self, d_ids, d_rows, n: int, d_n=None, d_mask=None, stream=None) -> None:
        if n <= 0:
            return
        if d_mask is None:
            rc = L.lib().bp_store_write(self.handle, L.ptr(d_ids), L.ptr(d_rows), n, L.ptr(d_n),
                                        L.stream_ptr(stream))
        else:
            rc = L.lib().bp_store_write_masked(self.handle, L.ptr(d_ids), L.ptr(d_rows), L.ptr(d_mask), n,
                                               L.ptr(d_n), L.stream_ptr(stream))
        L.check(rc, "bp_store_write")

    # -- reference API --------------------------------------------------------
    def fetch(self, keys) -> np.ndarray:
        """Current values for unique sorted keys, in key order (a copy)."""
        if not len(keys):
            return np.zeros((0, self.schema.emb_dim), dtype=np.float32)
        with self._lock:
            self.fetch_calls += 1
            ids = self._ids(keys)
            arr = np.asarray(keys, dtype=np.int64).reshape(len(keys), 2)
            d_ids = L.to_device(ids)
            d_keys = L.to_device(pack_keys(arr[:, 0], arr[:, 1]))
            out = self.fetch_ids_async(d_ids, len(ids), d_keys=d_keys)
            return out.cpu().numpy()

    def write_back(self, keys, values) -> None:
        """Overwrite values for unique keys, atomically per call."""
        if not len(keys):
            return
        if len(set(map(tuple, keys))) != len(keys):
            raise StoreError("write_back keys must be unique")
        with self._lock:
            self.write_calls += 1
            ids = self._ids(keys)
            vals = np.ascontiguousarray(values, dtype=np.float32).reshape(len(keys), self.schema.emb_dim)
            self.write_ids_async(L.to_device(ids), L.to_device(vals), len(ids))
            torch.cuda.current_stream().synchronize()
            self.entries_written += len(keys)

    def table_view(self) -> np.ndarray:
        """The whole store as a (total_rows, emb_dim) view of pinned memory
        (write-back log folded in first)."""
        torch.cuda.synchronize()
        L.check(L.lib().bp_store_compact(self.handle, L.stream_ptr()), "bp_store_compact")
        torch.cuda.synchronize()
        return self._table

    def written_mask(self) -> np.ndarray:
        torch.cuda.synchronize()
        words = (self.schema.total_rows + 31) // 32
        addr = L.lib().bp_store_written_bitmap(self.handle)
        bits = L.to_host(_device_u32(addr, words))
        mask = np.unpackbits(bits.view(np.uint8), bitorder="little")[: self.schema.total_rows]
        return mask.astype(bool)

    def _keys_of_ids(self, ids: np.ndarray) -> list:
        t = np.searchsorted(self._base, ids, side="right") - 1
        return [EmbeddingKey(int(a), int(b)) for a, b in zip(t, ids - self._base[t])]

    def written_items(self):
        """All explicitly written entries, sorted by key."""
        ids = np.flatnonzero(self.written_mask())
        table = self.table_view()
        for key, g in zip(self._keys_of_ids(ids), ids):
            yield key, table[g].copy()

    def snapshot_digest(self) -> str:
        """blake2b-128 over every value in (table, row, component) order."""
        h = hashlib.blake2b(digest_size=16)
        h.update(memoryview(self.table_view()).cast("B"))
        return h.hexdigest()

    def diff(self, other: "ShardedStore", limit: int = 100) -> list:
        """First ``limit`` keys whose values differ between two stores."""
        if self.schema != other.schema:
            raise StoreError("cannot diff stores with different schemas")
        a, b = self.table_view(), other.table_view()
        out = []
        step = 1 << 20
        for lo in range(0, a.shape[0], step):
            rows = np.flatnonzero((a[lo:lo + step] != b[lo:lo + step]).any(axis=1)) + lo
            for g, key in zip(rows, self._keys_of_ids(rows)):
                out.append((key, a[g].copy(), b[g].copy()))
                if len(out) >= limit:
                    return out
        return out


def _device_u32(addr: int, count: int) -> torch.Tensor:
    from .device import _wrap_device

    return _wrap_device(addr, torch.uint32, count)


def write_store_dump(store: ShardedStore, path: str) -> int:
    """EMSTD1 dump of the written entries (reference store.py:204-216)."""
    schema = store.schema
    ids = np.flatnonzero(store.written_mask())
    table = store.table_view()
    t = np.searchsorted(store._base, ids, side="right") - 1
    rec = np.zeros(len(ids), dtype=np.dtype([("t", "<u4"), ("r", "<u8"), ("v", "<f4", (schema.emb_dim,))]))
    rec["t"] = t
    rec["r"] = ids - store._base[t]
    rec["v"] = table[ids]
    with open(path, "wb") as fh:
        fh.write(DUMP_MAGIC)
        fh.write(struct.pack("<III", schema.num_tables, schema.num_dense, schema.emb_dim))
        fh.write(struct.pack(f"<{schema.num_tables}Q", *schema.rows_per_table))
        fh.write(struct.pack("<QQ", store.seed & 0xFFFFFFFFFFFFFFFF, len(ids)))
        fh.write(rec.tobytes())
    return len(ids)


def read_store_dump(path: str) -> ShardedStore:
    """Rebuild a store from an EMSTD1 dump (for offline diffing)."""
    with open(path, "rb") as fh:
        if fh.read(len(DUMP_MAGIC)) != DUMP_MAGIC:
            raise TraceFormatError("bad store dump magic")
        num_tables, num_dense, emb_dim = struct.unpack("<III", fh.read(12))
        rows = struct.unpack(f"<{num_tables}Q", fh.read(8 * num_tables))
        seed, count = struct.unpack("<QQ", fh.read(16))
        dt = np.dtype([("t", "<u4"), ("r", "<u8"), ("v", "<f4", (emb_dim,))])
        buf = fh.read(dt.itemsize * count)
        if len(buf) != dt.itemsize * count:
            raise TraceFormatError("truncated store dump")
    schema = Schema(num_tables, rows, num_dense, emb_dim)
    store = ShardedStore(schema, 1, seed)
    rec = np.frombuffer(buf, dtype=dt)
    if count:
        keys = [EmbeddingKey(int(a), int(b)) for a, b in zip(rec["t"], rec["r"])]
        store.write_back(keys, np.ascontiguousarray(rec["v"]))
    return store
