"""Trainer-resident TTL cache in HBM (reference cache.py:31-286 API).

All state lives on the GPU (``csrc/cache.cu``): the key -> slot map, the
float32 row arena, TTL / dirty / used per slot and the free list.  This class
is the reference-shaped front end: EmbeddingKey lists and numpy arrays in,
copies out, the same exceptions at the same points.  The engine drives the
same native object through its device-side entry points (no host copies).
"""

from __future__ import annotations

import ctypes as C
import hashlib

import numpy as np
import torch

from . import _lib as L
from .device import DeviceSchema, _wrap_device
from .errors import CacheCapacityError, CacheOrderingError, ConfigurationError
from .traces import EmbeddingKey, unpack_keys


class DynamicCache:
    """Map key -> (value vector, ttl, dirty) bounded by an entry capacity."""

    def __init__(self, capacity: int, emb_dim: int, schema=None):
        if capacity < 1:
            raise ConfigurationError("cache capacity must be >= 1")
        if emb_dim < 1:
            raise ConfigurationError("emb_dim must be >= 1")
        self.capacity = capacity
        self.emb_dim = emb_dim
        self.completed_iteration = None
        self.schema = schema
        sc = DeviceSchema.get(schema).handle if schema is not None else None
        h = C.c_void_p()
        L.check(L.lib().bp_cache_create(L.Context.get().handle, sc, capacity, emb_dim, C.byref(h)),
                "bp_cache_create")
        self.handle = h
        v = L.CacheView()
        L.check(L.lib().bp_cache_get_view(h, C.byref(v)), "bp_cache_get_view")
        self._view = v
        self.values = _wrap_device(v.d_values, torch.float32, capacity * emb_dim).view(capacity, emb_dim)
        self.ttl = _wrap_device(v.d_ttl, torch.int64, capacity)
        self.dirty = _wrap_device(v.d_dirty, torch.uint8, capacity)
        self.used = _wrap_device(v.d_used, torch.uint8, capacity)
        self.slot_key = _wrap_device(v.d_slot_key, torch.uint64, capacity)
        self._ctx = L.Context.get()

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                L.lib().bp_cache_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    # -- counters ---------------------------------------------------------------
    def stats(self) -> L.CacheStats:
        st = L.CacheStats()
        L.check(L.lib().bp_cache_get_stats(self.handle, L.stream_ptr(), C.byref(st)), "bp_cache_get_stats")
        return st

    @property
    def insertions(self) -> int:
        return int(self.stats().insertions)

    @property
    def evictions(self) -> int:
        return int(self.stats().evictions)

    @property
    def peak_occupancy(self) -> int:
        return int(self.stats().peak_occupancy)

    def __len__(self) -> int:
        return int(self.stats().occupancy)

    # -- inspection -------------------------------------------------------------
    def _resident(self):
        used = self.used.cpu().numpy().astype(bool)
        slots = np.flatnonzero(used)
        keys = self.slot_key.cpu().numpy()[slots]
        return slots, keys

    def key_set(self) -> set:
        _, keys = self._resident()
        return set(unpack_keys(keys))

    def __contains__(self, key) -> bool:
        return self._slot_of([key], check=False)[0] >= 0

    def _slot_of(self, keys, check: bool = True, iteration=None) -> np.ndarray:
        d_keys = L.to_device(L.host_u64(keys))
        out = torch.empty(len(keys), dtype=torch.int32, device="cuda")
        L.check(L.lib().bp_cache_resolve(self.handle, L.ptr(d_keys), None, len(keys), None,
                                         -1 if iteration is None else iteration, L.ptr(out), L.stream_ptr()),
                "bp_cache_resolve")
        slots = out.cpu().numpy().astype(np.int64)
        if check:
            self._ctx.raise_pending()
        else:
            try:
                self._ctx.raise_pending()
            except Exception:
                pass
        return slots

    def ttl_of(self, key) -> int:
        slot = self._slot_of([key], check=False)[0]
        if slot < 0:
            raise KeyError(key)
        return int(self.ttl[int(slot)].item())

    def is_dirty(self, key) -> bool:
        slot = self._slot_of([key], check=False)[0]
        if slot < 0:
            raise KeyError(key)
        return bool(self.dirty[int(slot)].item())

    # -- maintenance role ---------------------------------------------------------
    def apply_prefetch(self, keys, values, ttls) -> None:
        """Insert fetched entries clean, with the TTL the plan assigned."""
        n = len(keys)
        if n == 0:
            return
        occupancy = len(self)
        if occupancy + n > self.capacity:
            raise CacheCapacityError(f"inserting {n} entries into {occupancy}/{self.capacity}")
        seen = set()
        for key in keys:
            if key in seen:
                raise CacheOrderingError(f"duplicate insert for {key!r}")
            seen.add(key)
        try:
            ttl_arr = np.asarray([ttls[k] for k in keys], dtype=np.int64)
        except KeyError as exc:
            raise CacheOrderingError(f"prefetched key {exc.args[0]!r} has no TTL") from None
        vals = np.ascontiguousarray(values, dtype=np.float32).reshape(n, self.emb_dim)
        d_keys = L.to_device(L.host_u64(keys))
        d_vals = L.to_device(vals)
        d_ttl = L.to_device(ttl_arr)
        L.check(L.lib().bp_cache_insert(self.handle, L.ptr(d_keys), None, L.ptr(d_vals), L.ptr(d_ttl), n, None, -1,
                                        L.stream_ptr()), "bp_cache_insert")
        self._ctx.raise_pending()

    def apply_ttl_updates(self, updates) -> None:
        """Replace TTLs of resident keys; an absent key is an ordering violation."""
        updates = list(updates)
        if not updates:
            return
        keys = [k for k, _ in updates]
        d_keys = L.to_device(L.host_u64(keys))
        d_ttl = L.to_device(np.asarray([t for _, t in updates], dtype=np.int64))
        L.check(L.lib().bp_cache_set_ttl(self.handle, L.ptr(d_keys), None, L.ptr(d_ttl), len(keys), None, -1,
                                         L.stream_ptr()), "bp_cache_set_ttl")
        self._ctx.raise_pending()

    # -- training role -------------------------------------------------------------
    def resolve_slots(self, keys, iteration=None) -> np.ndarray:
        """Slot indices; any miss raises CacheMissError(key, iteration)."""
        if not len(keys):
            return np.zeros(0, dtype=np.int64)
        return self._slot_of(list(keys), check=True, iteration=iteration)

    def values_at(self, slot_idx) -> np.ndarray:
        slots = np.asarray(slot_idx, dtype=np.int64)
        if slots.size == 0:
            return np.zeros((0, self.emb_dim), dtype=np.float32)
        d_slots = L.to_device(slots.astype(np.int32))
        out = torch.empty((slots.size, self.emb_dim), dtype=torch.float32, device="cuda")
        L.check(L.lib().bp_cache_gather(self.handle, L.ptr(d_slots), slots.size, None, L.ptr(out), L.stream_ptr()),
                "bp_cache_gather")
        return out.cpu().numpy()

    def lookup_batch(self, keys, iteration=None) -> np.ndarray:
        if not keys:
            return np.zeros((0, self.emb_dim), dtype=np.float32)
        return self.values_at(self.resolve_slots(keys, iteration))

    def update_rows(self, slot_idx, new_values, dirty_mask) -> None:
        slots = np.asarray(slot_idx, dtype=np.int64)
        if slots.size == 0:
            return
        d_slots = L.to_device(slots.astype(np.int32))
        d_vals = L.to_device(np.ascontiguousarray(new_values, dtype=np.float32).reshape(slots.size, self.emb_dim))
        d_mask = L.to_device(np.asarray(dirty_mask, dtype=np.uint8))
        L.check(L.lib().bp_cache_update(self.handle, L.ptr(d_slots), L.ptr(d_vals), L.ptr(d_mask), slots.size, None,
                                        L.stream_ptr()), "bp_cache_update")

    def write_local_update(self, key, new_value) -> None:
        slot = self._slot_of([key], check=False)[0]
        if slot < 0:
            raise CacheOrderingError(f"update for absent key {key!r}")
        self.update_rows([slot], np.asarray(new_value, dtype=np.float32)[None, :], np.ones(1, dtype=bool))

    # -- eviction -------------------------------------------------------------------
    def _release(self, completed: int, drain: bool):
        n_max = self.capacity
        keys = torch.empty(n_max, dtype=torch.uint64, device="cuda")
        rows = torch.empty((n_max, self.emb_dim), dtype=torch.float32, device="cuda")
        dirty = torch.empty(n_max, dtype=torch.uint8, device="cuda")
        count = torch.zeros(2, dtype=torch.int64, device="cuda")
        buf = L.EvictBuffers(L.ptr(keys), None, L.ptr(rows), L.ptr(dirty), L.ptr(count))
        L.check(L.lib().bp_cache_evict(self.handle, completed, 1 if drain else 0, C.byref(buf), n_max,
                                       L.stream_ptr()), "bp_cache_evict")
        self._ctx.raise_pending()
        n = int(count[0].item())
        if n == 0:
            return [], np.zeros((0, self.emb_dim), dtype=np.float32), np.zeros(0, dtype=bool)
        k = keys[:n].cpu().numpy()
        order = np.argsort(k, kind="stable")
        return (unpack_keys(k[order]), rows[:n].cpu().numpy()[order], dirty[:n].cpu().numpy()[order].astype(bool))

    def evict_expired_arrays(self, completed: int):
        """(key-sorted keys, values, dirty) of every entry with ttl <= completed."""
        if self.completed_iteration is not None and completed < self.completed_iteration:
            raise CacheOrderingError(
                f"completed iteration went backwards: {completed} < {self.completed_iteration}")
        self.completed_iteration = completed
        return self._release(completed, drain=False)

    def evict_expired(self, completed: int) -> list:
        keys, values, dirty = self.evict_expired_arrays(completed)
        return [(k, values[i], bool(dirty[i])) for i, k in enumerate(keys)]

    def drain_arrays(self):
        return self._release(0, drain=True)

    def drain(self) -> list:
        keys, values, dirty = self.drain_arrays()
        return [(k, values[i], bool(dirty[i])) for i, k in enumerate(keys)]

    # -- replica checks ---------------------------------------------------------------
    def content_checksum(self) -> int:
        """Order-independent 64-bit checksum of (key, ttl, dirty, value), on the GPU."""
        out = torch.zeros(1, dtype=torch.uint64, device="cuda")
        L.check(L.lib().bp_cache_checksum(self.handle, L.ptr(out), L.stream_ptr()), "bp_cache_checksum")
        return int(out.cpu().numpy()[0])

    def canonical_digest(self) -> str:
        """blake2b over key-sorted (table, row, ttl, dirty, value) entries
        (reference cache.py:274-286): the records are laid out as one <i8 x 4 +
        <f4 x D structured array, so a single update hashes the same bytes as
        the reference's per-entry updates."""
        slots, keys = self._resident()
        order = np.argsort(keys, kind="stable")
        slots, keys = slots[order], np.asarray(keys, dtype=np.uint64)[order]
        rec = np.zeros(keys.size, dtype=[("h", "<i8", (4,)), ("v", "<f4", (self.emb_dim,))])
        if keys.size:
            d_slots = torch.from_numpy(np.asarray(slots, dtype=np.int64)).cuda()
            rec["h"][:, 0] = (keys >> np.uint64(44)).astype(np.int64)
            rec["h"][:, 1] = (keys & np.uint64((1 << 44) - 1)).astype(np.int64)
            rec["h"][:, 2] = self.ttl[d_slots].cpu().numpy()
            rec["h"][:, 3] = self.dirty[d_slots].cpu().numpy()
            rec["v"] = self.values[d_slots].cpu().numpy()
        h = hashlib.blake2b(digest_size=16)
        h.update(rec.tobytes())
        return h.hexdigest()


__all__ = ["DynamicCache", "EmbeddingKey"]
