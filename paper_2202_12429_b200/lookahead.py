"""Oracle Cacher: lookahead cache planning on the GPU (reference lookahead.py:1-189).

Algorithm 1 of the paper.  The scalar part -- the window queue, the lookahead
L and its halving under pressure -- stays on the host exactly as in the
reference; the per-key part (``latest_tracker`` and the ``in_cache`` mirror)
is device state updated by ``bp_planner_refill`` / ``bp_planner_pop`` over a
batch's GPU-deduplicated unique keys (``csrc/planner.cu``).

A :class:`CachePlan` produced here keeps its lists on the device; ``prefetch``
and ``ttl_updates`` materialise Python lists only when read.
"""

from __future__ import annotations

import ctypes as C
from collections import deque
from typing import Iterable, Iterator

import numpy as np
import torch

from . import _lib as L
from .device import DevicePrep, DeviceSchema
from .errors import ConfigurationError, RecordParseError
from .traces import Batch, EmbeddingKey, unpack_keys

_TRACKED = 1
_MIRRORED = 2


class DevicePlan:
    """Plan buffers of one emission, resident in HBM."""

    def __init__(self, prep: DevicePrep, exact: bool = True):
        # exact: size buffers by U (one sync); else by the occurrence count,
        # an upper bound known on the host, so emission never blocks.
        u = prep.num_unique if exact else prep.n_occ
        self.prep = prep
        self.h_pending = None
        self.cap = u
        dev = "cuda"
        self.prefetch_keys = torch.empty(max(u, 1), dtype=torch.uint64, device=dev)
        self.prefetch_ids = torch.empty(max(u, 1), dtype=torch.uint32, device=dev)
        self.prefetch_ttls = torch.empty(max(u, 1), dtype=torch.int64, device=dev)
        self.ttl_k = torch.empty(max(u, 1), dtype=torch.int64, device=dev)
        self.evict_keys = torch.empty(max(u, 1), dtype=torch.uint64, device=dev)
        self.counts = torch.zeros(5, dtype=torch.int64, device=dev)
        self.h_counts = None

    def buffers(self) -> L.PlanBuffers:
        return L.PlanBuffers(L.ptr(self.prefetch_keys), L.ptr(self.prefetch_ids), L.ptr(self.prefetch_ttls),
                             L.ptr(self.ttl_k), L.ptr(self.evict_keys), None, L.ptr(self.counts))

    def read_counts(self) -> np.ndarray:
        if self.h_counts is None:
            if self.h_pending is not None:
                self.h_counts = self.h_pending.counts().numpy().copy()
            else:
                self.h_counts = self.counts.cpu().numpy()
        return self.h_counts

    @property
    def n_prefetch(self) -> int:
        return int(self.read_counts()[0])

    @property
    def n_evict(self) -> int:
        return int(self.read_counts()[1])


class CachePlan:
    """Per-iteration planner output (reference lookahead.py:20-35).

    ``prefetch`` is sorted by (table_id, row_id); ``ttl_updates`` holds one
    (key, ttl) pair per unique key of the batch in first-occurrence order.
    """

    __slots__ = ("iteration", "lookahead", "_prefetch", "_ttl_updates", "device")

    def __init__(self, iteration: int, prefetch=None, ttl_updates=None, lookahead: int = 0, device=None):
        self.iteration = iteration
        self.lookahead = lookahead
        self._prefetch = prefetch
        self._ttl_updates = ttl_updates
        self.device = device

    @property
    def prefetch(self) -> list:
        if self._prefetch is None:
            n = self.device.n_prefetch
            self._prefetch = unpack_keys(L.to_host(self.device.prefetch_keys, n)) if n else []
        return self._prefetch

    @prefetch.setter
    def prefetch(self, value):
        self._prefetch = value

    @property
    def ttl_updates(self) -> list:
        if self._ttl_updates is None:
            d = self.device
            u = d.prep.num_unique
            if u == 0:
                self._ttl_updates = []
            else:
                keys = unpack_keys(L.to_host(d.prep.tensor("d_uniq_key_k", torch.uint64, u)))
                ttls = L.to_host(d.ttl_k, u).tolist()
                self._ttl_updates = list(zip(keys, ttls))
        return self._ttl_updates

    @ttl_updates.setter
    def ttl_updates(self, value):
        self._ttl_updates = value

    @property
    def prefetch_count(self) -> int:
        return self.device.n_prefetch if self._prefetch is None else len(self._prefetch)

    def evict_keys(self) -> list:
        """The planner's evict set {e in batch : ttl(e) == iteration}, sorted."""
        n = self.device.n_evict
        return unpack_keys(L.to_host(self.device.evict_keys, n)) if n else []

    def ttl_map(self) -> dict:
        return dict(self.ttl_updates)

    def __eq__(self, other):
        if not isinstance(other, CachePlan):
            return NotImplemented
        return (self.iteration, self.prefetch, self.ttl_updates, self.lookahead) == (
            other.iteration, other.prefetch, other.ttl_updates, other.lookahead)

    def __repr__(self) -> str:
        return f"CachePlan(iteration={self.iteration}, lookahead={self.lookahead}, prefetch={self.prefetch_count})"


class LookaheadState:
    """Planner state: host window queue + device tracker/mirror (reference lookahead.py:38-52)."""

    def __init__(self, lookahead: int, cache_capacity: int, schema=None, num_ranks: int = 1, prep_provider=None):
        self.lookahead = lookahead
        self.cache_capacity = cache_capacity
        self.batch_queue: deque = deque()
        self.projected_occupancy = 0
        self.insertions = 0
        self.removals = 0
        self.peak_occupancy = 0
        self.peak_projected = 0
        self.schema = schema
        self.num_ranks = num_ranks
        self._preps: deque = deque()
        self._provider = prep_provider
        sc = DeviceSchema.get(schema).handle if schema is not None else None
        h = C.c_void_p()
        L.check(L.lib().bp_planner_create(L.Context.get().handle, sc, cache_capacity, C.byref(h)),
                "bp_planner_create")
        self.handle = h

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                L.lib().bp_planner_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def _prep(self, batch: Batch) -> DevicePrep:
        if self._provider is not None:
            return self._provider(batch)
        return DevicePrep.from_batch(batch, self.num_ranks, self.schema)

    def stats(self) -> L.PlannerStats:
        st = L.PlannerStats()
        L.check(L.lib().bp_planner_get_stats(self.handle, L.stream_ptr(), C.byref(st)), "bp_planner_get_stats")
        return st

    def _dump(self):
        return planner_dump(self.handle)

    @property
    def in_cache(self) -> set:
        keys, _, flags = self._dump()
        return set(unpack_keys(keys[(flags & _MIRRORED) != 0]))

    def mirror_keys_u64(self) -> np.ndarray:
        keys, _, flags = self._dump()
        return np.sort(keys[(flags & _MIRRORED) != 0])

    @property
    def latest_tracker(self) -> dict:
        keys, last, flags = self._dump()
        sel = (flags & _TRACKED) != 0
        return dict(zip(unpack_keys(keys[sel]), last[sel].tolist()))


def planner_dump(handle, stream=None):
    """(keys, last iteration, flags) of every key with planner state."""
    st = L.PlannerStats()
    L.check(L.lib().bp_planner_get_stats(handle, L.stream_ptr(stream), C.byref(st)), "bp_planner_get_stats")
    cap = max(1, int(st.tracked) + int(st.in_cache) + 1)
    keys = torch.empty(cap, dtype=torch.uint64, device="cuda")
    last = torch.empty(cap, dtype=torch.int64, device="cuda")
    flags = torch.empty(cap, dtype=torch.uint8, device="cuda")
    count = torch.zeros(1, dtype=torch.int64, device="cuda")
    d = L.PlannerDump(L.ptr(keys), L.ptr(last), L.ptr(flags), L.ptr(count))
    L.check(L.lib().bp_planner_dump(handle, C.byref(d), cap, L.stream_ptr(stream)), "bp_planner_dump")
    torch.cuda.synchronize()
    n = min(int(count.item()), cap)
    return L.to_host(keys, n), L.to_host(last, n), L.to_host(flags, n)


def new_state(lookahead: int, cache_capacity: int, **kw) -> LookaheadState:
    """Fresh planner state for a window of ``lookahead`` batches (current included)."""
    if lookahead < 1:
        raise ConfigurationError("lookahead must be >= 1")
    if cache_capacity < 1:
        raise ConfigurationError("cache_capacity must be >= 1")
    return LookaheadState(lookahead, cache_capacity, **kw)


def emit_next_plan(state: LookaheadState, source: Iterator[Batch], stream=None) -> CachePlan | None:
    """Refill the window, pop its front batch and emit that batch's plan
    (reference lookahead.py:64-110); None once source and window are empty."""
    queue = state.batch_queue
    lib = L.lib()
    sp = L.stream_ptr(stream)
    while len(queue) < state.lookahead:
        batch = next(source, None)
        if batch is None:
            break
        prep = state._prep(batch)
        queue.append(batch)
        state._preps.append(prep)
        L.check(lib.bp_planner_refill(state.handle, prep.handle, sp), "bp_planner_refill")
    if not queue:
        st = state.stats()
        state.projected_occupancy = int(st.tracked)
        state.peak_projected = max(state.peak_projected, state.projected_occupancy)
        return None
    batch = queue.popleft()
    prep = state._preps.popleft()
    plan_dev = DevicePlan(prep)
    L.check(lib.bp_planner_pop(state.handle, prep.handle, C.byref(plan_dev.buffers()), sp), "bp_planner_pop")
    st = state.stats()  # synchronises: counts of this emission are final
    state.projected_occupancy = int(st.last_projected)
    state.peak_projected = int(st.peak_projected)
    state.peak_occupancy = int(st.peak_occupancy)
    state.insertions = int(st.insertions)
    state.removals = int(st.removals)
    return CachePlan(batch.iteration, None, None, state.lookahead, device=plan_dev)


def adapt_on_pressure(state: LookaheadState) -> bool:
    """Halve L when projected occupancy exceeds capacity (never below 1)."""
    if state.projected_occupancy > state.cache_capacity and state.lookahead > 1:
        state.lookahead = max(1, state.lookahead // 2)
        return True
    return False


def plan_trace(source: Iterable[Batch], lookahead: int, cache_capacity: int, **kw) -> Iterator[CachePlan]:
    """Exactly one CachePlan per batch, in order."""
    state = new_state(lookahead, cache_capacity, **kw)
    it = iter(source)
    while (plan := emit_next_plan(state, it)) is not None:
        yield plan
        adapt_on_pressure(state)


def auto_lookahead(source_prefix: Iterable[Batch], cache_capacity: int, schema=None, prep_provider=None) -> int:
    """Largest prefix length whose union of unique keys fits in the cache.

    The union size is the device planner's tracked count after each refill
    (nothing is ever popped), one synchronisation per batch scanned.
    """
    if cache_capacity < 1:
        raise ConfigurationError("cache_capacity must be >= 1")
    scan = LookaheadState(1, cache_capacity, schema=schema, prep_provider=prep_provider)
    n = 0
    for batch in source_prefix:
        prep = scan._prep(batch)
        L.check(L.lib().bp_planner_refill(scan.handle, prep.handle, L.stream_ptr()), "bp_planner_refill")
        seen = int(scan.stats().tracked)
        if seen > cache_capacity:
            if n == 0:
                raise ConfigurationError(
                    f"first batch alone needs {seen} cache entries, capacity is {cache_capacity}")
            return n
        n += 1
    if n == 0:
        raise ConfigurationError("auto lookahead needs at least one batch")
    return n


def format_plan(plan: CachePlan) -> str:
    """``iter=<n> prefetch=<t:r,...> ttl=<t:r@ttl,...>``"""
    pf = ",".join(f"{k[0]}:{k[1]}" for k in plan.prefetch)
    tt = ",".join(f"{k[0]}:{k[1]}@{t}" for k, t in plan.ttl_updates)
    return f"iter={plan.iteration} prefetch={pf} ttl={tt}"


def parse_plan(line: str) -> CachePlan:
    """Inverse of :func:`format_plan`; the lookahead is not serialized and reads 0."""
    try:
        it_part, pf_part, ttl_part = line.strip().split(" ")
        iteration = int(it_part.removeprefix("iter="))
        pf_body = pf_part.removeprefix("prefetch=")
        ttl_body = ttl_part.removeprefix("ttl=")
        prefetch = [EmbeddingKey(*map(int, tok.split(":"))) for tok in pf_body.split(",")] if pf_body else []
        ttl_updates = []
        if ttl_body:
            for tok in ttl_body.split(","):
                kpart, ttl = tok.split("@")
                t, r = kpart.split(":")
                ttl_updates.append((EmbeddingKey(int(t), int(r)), int(ttl)))
    except (ValueError, TypeError):
        raise RecordParseError(f"bad plan record: {line!r}") from None
    return CachePlan(iteration, prefetch, ttl_updates, 0)
