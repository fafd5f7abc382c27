"""Device-resident objects behind the reference API: schemas and batch preps.

A :class:`DevicePrep` is one batch uploaded to HBM and grouped by key on the
GPU (``bp_prep_create``): the replacement for ``Batch.unique_keys`` and
``_prep_batch`` (reference traces.py:91-103, engine.py:142-182).  It owns the
uploaded key/label tensors until the prep is destroyed, so stream ordering
alone keeps the kernels' inputs alive.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L
from .traces import Batch, Schema, unpack_keys


class DeviceSchema:
    """bp_schema: table cardinalities + dense-id bases in HBM."""

    _cache: dict = {}

    def __init__(self, schema: Schema):
        self.schema = schema
        rows = np.ascontiguousarray(schema.rows_per_table, dtype=np.int64)
        h = C.c_void_p()
        L.check(L.lib().bp_schema_create(schema.num_tables, rows.ctypes.data, schema.emb_dim, C.byref(h)),
                "bp_schema_create")
        self.handle = h
        self.total_rows = schema.total_rows

    @classmethod
    def get(cls, schema: Schema) -> "DeviceSchema":
        ds = cls._cache.get(schema)
        if ds is None:
            ds = cls(schema)
            cls._cache[schema] = ds
        return ds

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                L.lib().bp_schema_destroy(self.handle)
        except Exception:
            pass


class Uploader:
    """Host -> HBM batch uploads through a ring of reusable pinned buffers.

    ``tensor.pin_memory()`` per batch costs a pinned allocation each time; the
    ring copies the numpy batch into a pre-pinned slot (waiting only for that
    slot's previous DMA) and issues one asynchronous H2D copy.
    """

    def __init__(self, slot_bytes: int, slots: int = 4):
        self.slot_bytes = slot_bytes
        self.bufs = [torch.empty(slot_bytes, dtype=torch.uint8, pin_memory=True) for _ in range(slots)]
        self.views = [b.numpy() for b in self.bufs]
        self.events = [None] * slots
        self.i = 0

    def upload(self, arr: np.ndarray, stream) -> torch.Tensor:
        arr = np.ascontiguousarray(arr)
        nbytes = arr.nbytes
        if nbytes > self.slot_bytes:
            return L.to_device(arr, stream)
        k = self.i
        self.i = (self.i + 1) % len(self.bufs)
        if self.events[k] is not None:
            self.events[k].synchronize()
        view = self.views[k][:nbytes]
        view[:] = arr.view(np.uint8).reshape(-1)
        out = torch.empty(arr.shape, dtype=_TORCH_OF[arr.dtype.str], device="cuda")
        with torch.cuda.stream(stream):
            out.view(torch.uint8).reshape(-1).copy_(self.bufs[k][:nbytes], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        self.events[k] = ev
        return out


_TORCH_OF = {"<u8": torch.uint64, "|u1": torch.uint8, "<i8": torch.int64, "<u4": torch.uint32, "<f4": torch.float32}


def _bits(x: int) -> int:
    return max(1, int(x).bit_length())


class DevicePrep:
    """One batch on the GPU: uniques (sorted and first-occurrence), per-key
    occurrence lists, labels, trainer-rank bounds."""

    def __init__(self, keys: np.ndarray, labels: np.ndarray, rank_bounds: np.ndarray, iteration: int,
                 schema: Schema | None = None, occ_index: int = 0, stream=None,
                 d_keys: torch.Tensor | None = None, d_labels: torch.Tensor | None = None, uploader=None,
                 columns=None):
        lib = L.lib()
        self.stream = stream or torch.cuda.current_stream()
        self.n_occ = int(len(keys)) if d_keys is None else int(d_keys.numel())
        self.iteration = int(iteration)
        self.num_ranks = len(rank_bounds) - 1
        self.schema = schema
        up = uploader.upload if uploader is not None else L.to_device
        self.d_keys = d_keys if d_keys is not None else up(np.asarray(keys, dtype=np.uint64), self.stream)
        self.d_labels = d_labels if d_labels is not None else up(np.asarray(labels, dtype=np.uint8), self.stream)
        rb = np.ascontiguousarray(rank_bounds, dtype=np.int64)
        row_bits = table_bits = 1
        if schema is None and self.n_occ:
            k = np.asarray(keys, dtype=np.uint64)
            row_bits = _bits(int((k & np.uint64((1 << 44) - 1)).max()))
            table_bits = _bits(int((k >> np.uint64(44)).max()))
        sc = DeviceSchema.get(schema).handle if schema is not None else None
        h = C.c_void_p()
        if columns is not None and schema is not None:
            # Criteo layout (one key per table per example): per-column sort
            n_ex, tables = columns
            self.d_tables = L.to_device(np.ascontiguousarray(tables, dtype=np.int32), self.stream)
            L.check(lib.bp_prep_create_columnar(L.Context.get().handle, sc, L.ptr(self.d_keys), L.ptr(self.d_labels),
                                                n_ex, len(tables), L.ptr(self.d_tables), rb.ctypes.data,
                                                self.num_ranks, self.iteration, int(occ_index),
                                                L.stream_ptr(self.stream), C.byref(h)), "bp_prep_create_columnar")
        else:
            L.check(lib.bp_prep_create(L.Context.get().handle, sc, L.ptr(self.d_keys), L.ptr(self.d_labels),
                                       self.n_occ, rb.ctypes.data, self.num_ranks, self.iteration,
                                       int(occ_index), row_bits, table_bits, L.stream_ptr(self.stream),
                                       C.byref(h)), "bp_prep_create")
        self.handle = h
        v = L.PrepView()
        L.check(lib.bp_prep_get_view(h, C.byref(v)), "bp_prep_get_view")
        self.view = v
        self._num_unique = None

    @classmethod
    def from_batch(cls, batch: Batch, num_ranks: int = 1, schema: Schema | None = None, occ_index: bool = False,
                   stream=None, uploader=None) -> "DevicePrep":
        keys, labels, _ = batch.packed_occurrences()
        columns = None
        if schema is not None and batch.is_columnar and batch.num_examples:
            tables = batch.table_ids()
            if bool(np.all(np.diff(tables) > 0)):
                columns = (batch.num_examples, tables)
        return cls(keys, labels, batch.rank_bounds(num_ranks), batch.iteration, schema, occ_index, stream,
                   uploader=uploader, columns=columns)

    @property
    def num_unique(self) -> int:
        """U (synchronises once)."""
        if self._num_unique is None:
            out = C.c_int64()
            L.check(L.lib().bp_prep_num_unique(self.handle, L.stream_ptr(self.stream), C.byref(out)),
                    "bp_prep_num_unique")
            self._num_unique = int(out.value)
        return self._num_unique

    def tensor(self, name: str, dtype, count: int) -> torch.Tensor:
        """Zero-copy torch view of one device array of the prep."""
        addr = getattr(self.view, name)
        return _wrap_device(addr, dtype, count)

    def unique_keys_first(self) -> list:
        u = self.num_unique
        return unpack_keys(L.to_host(self.tensor("d_uniq_key_k", torch.uint64, u)))

    def unique_keys_sorted_u64(self) -> np.ndarray:
        return L.to_host(self.tensor("d_uniq_key_s", torch.uint64, self.num_unique))

    def destroy(self):
        if getattr(self, "handle", None):
            L.lib().bp_prep_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


_DTYPE_SIZE = {torch.uint64: 8, torch.int64: 8, torch.uint32: 4, torch.int32: 4, torch.uint8: 1, torch.float32: 4}


_CARRIER = {torch.uint64: (torch.int64, "<i8"), torch.int64: (torch.int64, "<i8"),
            torch.uint32: (torch.int32, "<i4"), torch.int32: (torch.int32, "<i4"),
            torch.uint8: (torch.uint8, "|u1"), torch.float32: (torch.float32, "<f4")}


class _CudaArrayInterface:
    def __init__(self, addr: int, typestr: str, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (addr, False),
                                         "version": 3, "strides": None}


def _wrap_device(addr: int, dtype: torch.dtype, count: int) -> torch.Tensor:
    """Non-owning tensor over native device memory (signed carrier, then a
    same-width dtype view, so unsigned types need no CAI support)."""
    if count == 0 or not addr:
        return torch.empty(0, dtype=dtype, device="cuda")
    carrier, typestr = _CARRIER[dtype]
    t = torch.as_tensor(_CudaArrayInterface(addr, typestr, count), device="cuda")
    return t if carrier == dtype else t.view(dtype)
