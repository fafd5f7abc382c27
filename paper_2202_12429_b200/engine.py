"""Pipelined BagPipe engine and synchronous oracle, executed on the GPU.

API of reference engine.py:42-825 (``EngineConfig``, ``run_pipeline``,
``run_synchronous_baseline``, ``verify_equivalence``).  The control flow --
dispatch gate, forced flushes, batched round-robin write-back, simulated
clock, report -- is host arithmetic that follows reference engine.py:239-672
step for step, so reports are byte-identical.  Every per-key operation runs
on the device:

  plan emission   bp_planner_refill / bp_planner_pop        (csrc/planner.cu)
  prefetch        bp_store_fetch: zero-copy gather from the pinned table
  apply + lookup  bp_cache_insert + bp_cache_apply_resolve  (csrc/cache.cu)
  train           bp_stub_step: gradient, rank-ordered combine, SGD, dirty,
                  critical-set count, fused                 (csrc/trainer.cu)
  maintenance     bp_cache_evict (ttl <= x) into a device flush chunk
  write-back      bp_store_write_masked: zero-copy scatter of dirty rows

The T data-parallel trainers of the reference hold identical cache
replicas (engine.py:267, 526-528).  On one GPU they collapse into one
physical cache: T survives as the rank split of every batch, i.e. the
accumulation order of the gradient combine, which is all that reaches the
digest.  One host synchronisation per iteration reads the counters the
report and the gate need.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import math
from bisect import bisect_right
from collections import deque
from dataclasses import asdict, dataclass, field
from typing import Iterable

import numpy as np
import torch

from . import _lib as L
from .cache import DynamicCache
from .device import DevicePrep, Uploader
from .errors import CacheCapacityError, ConfigurationError, EngineError, IncomparableRunsError
from .lookahead import CachePlan, DevicePlan, adapt_on_pressure, auto_lookahead, new_state
from .report import IterationRecord, RunReport
from .store import ShardedStore
from .trainer import BP_STUB_SGD, StubModelConfig, f32
from .traces import Batch, Schema, unpack_key, unpack_keys

_MODES = ("serial", "threaded")
FAULT_NO_GATE = "no_gate"
FAULT_DROP_PREFETCH = "drop_prefetch"


@dataclass
class EngineConfig:
    """Knobs for one run; mirrors the JSON config file field for field."""

    cache_capacity: int
    batch_size: int
    lookahead: int = 0
    num_trainers: int = 1
    num_shards: int = 1
    rpc_batch_proportion: float = 0.25
    fetch_latency: float = 0.25
    compute_latency: float = 1.0
    sync_bandwidth: float = 1000.0
    lr: float = 0.01
    c_value: float = 0.01
    c_label: float = 0.001
    seed: int = 0
    iterations: int = 0
    split_sync: bool = True
    mode: str = "serial"
    replication_check_interval: int = 64
    check_mirror: bool = False
    record_events: bool = False

    def __post_init__(self):
        checks = (
            (self.cache_capacity >= 1, "cache_capacity must be >= 1"),
            (self.batch_size >= 1, "batch_size must be >= 1"),
            (self.lookahead >= 0, "lookahead must be >= 0 (0 = auto)"),
            (self.num_trainers >= 1, "num_trainers must be >= 1"),
            (0 < self.rpc_batch_proportion <= 1, "rpc_batch_proportion must be in (0, 1]"),
            (self.fetch_latency >= 0 and self.compute_latency >= 0, "latencies must be >= 0"),
            (self.sync_bandwidth > 0, "sync_bandwidth must be > 0"),
            (self.iterations >= 0, "iterations must be >= 0"),
            (self.mode in _MODES, f"mode must be one of {_MODES}"),
            (self.replication_check_interval >= 1, "replication_check_interval must be >= 1"),
        )
        for ok, msg in checks:
            if not ok:
                raise ConfigurationError(msg)

    def stub(self) -> StubModelConfig:
        return StubModelConfig(lr=self.lr, c_value=self.c_value, c_label=self.c_label)

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, data: dict) -> "EngineConfig":
        unknown = set(data) - set(cls.__dataclass_fields__)
        if unknown:
            raise ConfigurationError(f"unknown config fields: {sorted(unknown)}")
        return cls(**data)


def load_config(path: str) -> EngineConfig:
    with open(path, "r", encoding="utf-8") as fh:
        return EngineConfig.from_dict(json.load(fh))


def _schema_dict(schema: Schema) -> dict:
    return {"num_tables": schema.num_tables, "rows_per_table": list(schema.rows_per_table),
            "num_dense": schema.num_dense, "emb_dim": schema.emb_dim}


def _materialize(trace: Iterable[Batch], iterations: int) -> list:
    batches = list(trace)
    if iterations > 0:
        batches = batches[:iterations]
    if not batches:
        raise ConfigurationError("trace has no batches")
    base = batches[0].iteration
    for i, b in enumerate(batches):
        if b.iteration != base + i:
            raise EngineError(f"batch iterations not consecutive at position {i}")
    return batches


def _totals(records: list) -> dict:
    return {
        "compute_time": sum(r.compute for r in records),
        "critical_sync_time": sum(r.critical_sync for r in records),
        "blocked_on_prefetch": sum(r.blocked_on_prefetch for r in records),
        "blocked_on_eviction": sum(r.blocked_on_eviction for r in records),
        "blocked_on_background": sum(r.blocked_on_background for r in records),
        "churn": sum(r.churn for r in records),
        "critical_entries": sum(r.critical_size for r in records),
        "background_entries": sum(r.background_size for r in records),
    }


_METADATA = {
    "clean_eviction_writeback": "skipped",
    "cache_sync_semantics": "gradient-sum-local-apply",
    "background_apply": "before-eviction-capture",
    "flush_rotation": "round-robin",
    "clock": "simulated",
}


class _Chunk:
    """Evictions of one iteration, still in HBM, awaiting a flush."""

    __slots__ = ("ids", "rows", "dirty", "count", "n", "n_dirty", "keys")

    def __init__(self, ids, rows, dirty, count, keys=None):
        self.ids, self.rows, self.dirty, self.count, self.keys = ids, rows, dirty, count, keys
        self.n = self.n_dirty = 0


class _PendingPlan:
    """An emitted plan whose device counters are read lazily (the next host
    synchronisation makes them final), so emission never blocks the host."""

    __slots__ = ("plan", "h_counts", "done")

    def __init__(self, plan, stream):
        self.plan = plan
        self.h_counts = torch.empty(4, dtype=torch.int64, pin_memory=True)
        self.h_counts.copy_(plan.device.counts, non_blocking=True)
        self.done = torch.cuda.Event()
        self.done.record(stream)

    def counts(self):
        if not self.done.query():
            self.done.synchronize()
        return self.h_counts


class _Pipeline:
    """One pipelined run (reference engine.py:239-649) driving the GPU.

    ``begin`` / ``step(pos)`` / ``end`` split the reference's run loop so a
    benchmark can time single iterations.  Each step enqueues its kernels
    with device-side counts and synchronises exactly once, at the end, to
    read the counters the simulated clock, the gate and the report need.
    """

    def __init__(self, cfg: EngineConfig, schema: Schema, batches: list, fingerprint, fault, device_inputs=None):
        if fault not in (None, FAULT_NO_GATE, FAULT_DROP_PREFETCH):
            raise ConfigurationError(f"unknown fault {fault!r}")
        self.cfg, self.schema, self.batches = cfg, schema, batches
        self.fingerprint, self.fault = fingerprint, fault
        self.base = batches[0].iteration
        self.n = len(batches)
        self.T = cfg.num_trainers
        self.stream = torch.cuda.current_stream()
        # Host-link traffic (prefetch gathers, write-back scatters) runs on its
        # own stream so it overlaps the compute of the current iteration; the
        # gate order of reference engine.py:302-377 is kept by issuing both in
        # dispatch order on that one stream, fenced by events.
        self.link = torch.cuda.Stream()
        self.device_inputs = device_inputs  # optional {pos: (d_keys, d_labels)} already in HBM
        self._preps: dict = {}
        self._uploader = None
        stub = cfg.stub()
        self.c_value, self.c_label, self.lr = f32(stub.c_value), f32(stub.c_label), f32(stub.lr)
        self.probe = None  # optional callable(name, phase) for kernel timing

        self.L0 = cfg.lookahead or auto_lookahead(iter(batches), cfg.cache_capacity, schema=schema,
                                                  prep_provider=self._prep_of_batch)
        self.flush_interval = max(1, math.ceil(cfg.rpc_batch_proportion * self.L0))
        self.store = ShardedStore(schema, cfg.num_shards, cfg.seed)
        self.cache = DynamicCache(cfg.cache_capacity, schema.emb_dim, schema=schema)
        self.occupancy = 0
        self.state = new_state(self.L0, cfg.cache_capacity, schema=schema, num_ranks=self.T,
                               prep_provider=self._prep_of_batch)
        self.source = iter(batches)
        self.snapshots = {} if cfg.check_mirror else None
        self._adapt_pending = None

        self.pending: deque = deque()
        self.exhausted = False
        self.staged: dict = {}
        self.chunks: list = []
        self.min_unflushed_ttl = None
        self.flushed_through = self.base - 1
        self.event_starts: list = []
        self.event_completes: list = []
        self.flush_log: list = []
        self.flush_counter = 0
        self.forced_flushes = 0
        self.crit_end = 0.0
        self.bg_end = 0.0
        self.records: list = []
        self.events = [] if cfg.record_events else None
        self.clean_evictions = 0
        self.dirty_evictions = 0
        self.total_prefetched = 0
        self.peak_occupancy = 0
        self.drop_done = False
        self.stats = torch.zeros(2, dtype=torch.int64, device="cuda")
        # dense per-row stamp of the next batch's keys (critical-set test)
        self.mark = torch.full((schema.total_rows,), -(1 << 62), dtype=torch.int64, device="cuda")
        self.h_step = torch.zeros(8, dtype=torch.int64, pin_memory=True)
        self.kernel_launches = 0

    # -- batch preps (device) ------------------------------------------------------
    def _prep_of_batch(self, batch: Batch) -> DevicePrep:
        pos = batch.iteration - self.base
        prep = self._preps.get(pos)
        if prep is None:
            dev = self.device_inputs.get(pos) if self.device_inputs else None
            if dev is not None:
                keys, labels = dev
                n = keys.numel()
                prep = DevicePrep(None, None, batch.rank_bounds(self.T), batch.iteration, self.schema,
                                  stream=self.stream, d_keys=keys, d_labels=labels)
            else:
                if self._uploader is None:
                    occ = batch.packed_occurrences()[0].size
                    self._uploader = Uploader(max(1 << 20, 16 * occ), slots=8)
                prep = DevicePrep.from_batch(batch, self.T, self.schema, stream=self.stream, uploader=self._uploader)
            self._preps[pos] = prep
        return prep

    def _prep(self, pos: int) -> DevicePrep:
        return self._prep_of_batch(self.batches[pos])

    # -- plan emission (reference engine.py:198-236, lookahead.py:64-123) --------
    def _next_plan(self):
        st = self.state
        if self._adapt_pending is not None:
            # The reference adapts lazily, when the next plan is requested.
            st.projected_occupancy = int(self._adapt_pending.counts()[2])
            adapt_on_pressure(st)
            self._adapt_pending = None
        lib = L.lib()
        sp = L.stream_ptr(self.stream)
        while len(st.batch_queue) < st.lookahead:
            batch = next(self.source, None)
            if batch is None:
                break
            prep = self._prep_of_batch(batch)
            st.batch_queue.append(batch)
            st._preps.append(prep)
            L.check(lib.bp_planner_refill(st.handle, prep.handle, sp), "bp_planner_refill")
        if not st.batch_queue:
            return None
        batch = st.batch_queue.popleft()
        prep = st._preps.popleft()
        dev = DevicePlan(prep, exact=False)
        L.check(lib.bp_planner_pop(st.handle, prep.handle, C.byref(dev.buffers()), sp), "bp_planner_pop")
        plan = CachePlan(batch.iteration, None, None, st.lookahead, device=dev)
        self._adapt_pending = _PendingPlan(plan, self.stream)
        dev.h_pending = self._adapt_pending
        if self.snapshots is not None:
            self.snapshots[plan.iteration - self.base] = st.mirror_keys_u64()
        return plan

    def _dispatch_pos(self, plan) -> int:
        pos = plan.iteration - self.base
        s = pos - plan.lookahead
        if s < 0:
            return -1
        if self.fault == FAULT_NO_GATE:
            return s
        p = self.flush_interval
        return min(((s + p) // p) * p - 1, pos - 1)

    def _gate_time(self, theta: int) -> float:
        j = bisect_right(self.event_starts, theta) - 1
        return self.event_completes[j] if j >= 0 else 0.0

    def _dispatch(self, plan, cur: int) -> None:
        theta = plan.iteration - plan.lookahead
        if self.fault != FAULT_NO_GATE and self.min_unflushed_ttl is not None and self.min_unflushed_ttl <= theta:
            self._flush("forced", cur)
            self.forced_flushes += 1
        arrival = self._gate_time(theta) + self.cfg.fetch_latency
        dev = plan.device
        self.link.wait_event(dev.h_pending.done)  # the plan's pop has run
        self._probe("store_fetch", 0, self.link)
        rows = self.store.fetch_ids_async(dev.prefetch_ids, dev.cap, d_n=dev.counts[0:1], stream=self.link)
        self._probe("store_fetch", 1, self.link)
        for t in (rows, dev.prefetch_ids, dev.counts):
            t.record_stream(self.link)
        fetched = torch.cuda.Event()
        fetched.record(self.link)
        self.staged[plan.iteration - self.base] = (plan, rows, arrival, fetched)

    def _dispatch_until(self, cur: int) -> None:
        while True:
            if not self.pending:
                if self.exhausted:
                    return
                plan = self._next_plan()
                if plan is None:
                    self.exhausted = True
                    return
                self.pending.append(plan)
            plan = self.pending[0]
            if self._dispatch_pos(plan) > cur:
                return
            self.pending.popleft()
            self._dispatch(plan, cur)

    def _probe(self, name: str, phase: int, stream=None) -> None:
        if self.probe is not None:
            self.probe(name, phase, stream or self.stream)

    # -- write-back (reference engine.py:350-377) ---------------------------------
    def _flush(self, kind: str, pos: int) -> None:
        flusher = self.flush_counter % self.T
        count = 0
        if self.chunks:
            # Chunks were produced on the compute stream, which the host has
            # synchronised since; the scatter runs on the link stream.
            self._probe("store_write", 0, self.link)
            for ch in self.chunks:  # in eviction order: the last write wins
                self.store.write_ids_async(ch.ids, ch.rows, ch.n, d_mask=ch.dirty, stream=self.link)
                for t in (ch.ids, ch.rows, ch.dirty):
                    t.record_stream(self.link)
            self._probe("store_write", 1, self.link)
            count = self._merged_count()
            self.store.write_calls += 1
            self.store.entries_written += count
        self.event_starts.append(self.flushed_through + 1)
        self.event_completes.append(max(self.crit_end, self.bg_end) + self.cfg.fetch_latency)
        self.flush_log.append({"position": pos, "kind": kind, "entries": count, "trainer": flusher})
        self.flushed_through = self.base + pos
        self.min_unflushed_ttl = None
        self.chunks = []
        self.flush_counter += 1

    def _merged_count(self) -> int:
        if len(self.chunks) == 1 or self.fault != FAULT_NO_GATE:
            # Under the gate a key cannot be evicted twice within one flush
            # window (its re-prefetch waits for the flush of the first
            # eviction), so chunk key sets are disjoint.
            return sum(ch.n_dirty for ch in self.chunks)
        ids = [L.to_host(ch.ids, ch.n)[L.to_host(ch.dirty, ch.n).astype(bool)] for ch in self.chunks]
        return int(np.unique(np.concatenate(ids)).size)

    # -- per iteration ---------------------------------------------------------------
    def _evict(self, completed: int, drain: bool, out_cap: int) -> _Chunk:
        cap = max(1, out_cap)
        dim = self.schema.emb_dim
        ch = _Chunk(torch.empty(cap, dtype=torch.uint32, device="cuda"),
                    torch.empty((cap, dim), dtype=torch.float32, device="cuda"),
                    torch.empty(cap, dtype=torch.uint8, device="cuda"),
                    torch.zeros(2, dtype=torch.int64, device="cuda"),
                    torch.empty(cap, dtype=torch.uint64, device="cuda") if self.events is not None else None)
        buf = L.EvictBuffers(L.ptr(ch.keys), L.ptr(ch.ids), L.ptr(ch.rows), L.ptr(ch.dirty), L.ptr(ch.count))
        L.check(L.lib().bp_cache_evict(self.cache.handle, completed, 1 if drain else 0, C.byref(buf), cap,
                                       L.stream_ptr(self.stream)), "bp_cache_evict")
        return ch

    def _buffer(self, ch: _Chunk, iteration: int) -> None:
        self.clean_evictions += ch.n - ch.n_dirty
        self.dirty_evictions += ch.n_dirty
        if ch.n_dirty:
            self.chunks.append(ch)
            if self.min_unflushed_ttl is None or iteration < self.min_unflushed_ttl:
                self.min_unflushed_ttl = iteration

    def _sorted_keys(self, ch: _Chunk) -> list:
        if ch.keys is None or ch.n == 0:
            return []
        return unpack_keys(np.sort(L.to_host(ch.keys, ch.n)))

    def begin(self) -> None:
        self._dispatch_until(-1)

    def step(self, pos: int) -> None:
        cfg, lib, ctx = self.cfg, L.lib(), L.Context.get()
        sp = L.stream_ptr(self.stream)
        bw = cfg.sync_bandwidth
        batch = self.batches[pos]
        if pos > 0:
            self._dispatch_until(pos - 1)
        iteration = batch.iteration
        staged = self.staged.pop(pos, None)
        if staged is None:
            raise EngineError(f"no staged prefetch for position {pos}")
        plan, rows, arrival, fetched = staged
        if plan.iteration != iteration:
            raise EngineError(f"plan {plan.iteration} misaligned with batch {iteration}")
        dev = plan.device
        prep = self._prep(pos)
        self.stream.wait_event(fetched)
        off, skip_key, has_skip = 0, 0, 0
        if self.fault == FAULT_DROP_PREFETCH and not self.drop_done and pos >= self.n // 2 and dev.n_prefetch:
            # Drop the first (smallest) prefetched key: it is neither inserted
            # nor TTL-updated, so the lookup must miss (reference engine.py:512-523).
            skip_key = int(L.to_host(dev.prefetch_keys, 1)[0])
            has_skip, off = 1, 1
            self.drop_done = True
        dim = self.schema.emb_dim
        # apply_prefetch: device count (minus the dropped key), device-side capacity check
        if off:
            n_ins_dev = dev.counts[0:1] - off
        else:
            n_ins_dev = dev.counts[0:1]
        self._probe("cache_insert", 0)
        L.check(lib.bp_cache_insert(
            self.cache.handle, L.ptr(dev.prefetch_keys) + 8 * off, L.ptr(dev.prefetch_ids) + 4 * off,
            L.ptr(rows) + 4 * dim * off, L.ptr(dev.prefetch_ttls) + 8 * off, max(dev.cap - off, 0),
            L.ptr(n_ins_dev), iteration, sp), "bp_cache_insert")
        slots = torch.empty(max(prep.n_occ, 1), dtype=torch.int32, device="cuda")
        L.check(lib.bp_cache_apply_resolve(self.cache.handle, prep.handle, L.ptr(dev.ttl_k), skip_key, has_skip,
                                           L.ptr(slots), sp), "bp_cache_apply_resolve")
        self._probe("cache_insert", 1)
        nxt = self._prep(pos + 1) if pos + 1 < self.n else None
        if nxt is not None:
            L.check(lib.bp_mark_ids(nxt.handle, L.ptr(self.mark), nxt.iteration, sp), "bp_mark_ids")
        self.stats.zero_()
        self._probe("stub_step", 0)
        L.check(lib.bp_stub_step(ctx.handle, prep.handle, L.ptr(self.cache.values), L.ptr(slots),
                                 L.ptr(self.cache.dirty), dim, self.c_value, self.c_label, self.lr, BP_STUB_SGD, None,
                                 L.ptr(self.mark) if nxt is not None else None,
                                 nxt.iteration if nxt is not None else 0, L.ptr(self.stats), sp), "bp_stub_step")
        self._probe("stub_step", 1)
        self._probe("cache_evict", 0)
        ch = self._evict(iteration, False, min(cfg.cache_capacity, max(prep.n_occ, 1)))
        self._probe("cache_evict", 1)
        # one host synchronisation: counters for the clock, gate and report
        h = self.h_step
        h[0:1].copy_(prep.tensor("d_num_unique", torch.int64, 1), non_blocking=True)
        h[1:2].copy_(n_ins_dev, non_blocking=True)
        h[2:4].copy_(self.stats, non_blocking=True)
        h[4:6].copy_(ch.count, non_blocking=True)
        ctx.raise_pending(self.stream)
        u, n_ins, crit_count, _, n_ev, n_ev_dirty = (int(v) for v in h[:6].tolist())
        ch.n, ch.n_dirty = n_ev, n_ev_dirty
        self.occupancy += n_ins
        occupancy_peak = self.occupancy
        self.occupancy -= n_ev
        self.peak_occupancy = max(self.peak_occupancy, occupancy_peak)
        self.total_prefetched += n_ins
        if n_ins:
            self.store.fetch_calls += 1

        stall = max(0.0, arrival - self.crit_end)
        blocked_prefetch = min(stall, max(0.0, cfg.fetch_latency - self.crit_end))
        blocked_eviction = stall - blocked_prefetch
        compute_end = self.crit_end + stall + cfg.compute_latency
        if cfg.split_sync:
            critical_size = crit_count if nxt is not None else 0
            background_size = u - critical_size
        else:
            critical_size, background_size = u, 0
        sync_start = max(compute_end, self.bg_end)
        blocked_background = sync_start - compute_end
        self.crit_end = sync_start + critical_size / bw
        self.bg_end = self.crit_end + background_size / bw
        partial = {
            "iteration": iteration, "warmup": pos < self.L0, "compute": cfg.compute_latency,
            "critical_sync": critical_size / bw, "blocked_on_prefetch": blocked_prefetch,
            "blocked_on_eviction": blocked_eviction, "blocked_on_background": blocked_background,
            "occupancy_peak": occupancy_peak, "prefetch_count": n_ins, "critical_size": critical_size,
            "background_size": background_size, "lookahead": plan.lookahead,
        }
        if self.events is not None:
            ttl = plan.ttl_updates
            if has_skip:
                lost = unpack_key(skip_key)
                ttl = [(k, t) for k, t in ttl if k != lost]
            partial["prefetch_keys"] = list(plan.prefetch[off:])
            partial["ttl_updates"] = list(ttl)
        self._maintenance(pos, ch, partial)
        self._preps.pop(pos, None)

    def end(self) -> RunReport:
        if not self.exhausted and (self.pending or self._next_plan() is not None):
            raise EngineError("planner emitted more plans than batches")
        return self._report()

    def run(self) -> RunReport:
        self.begin()
        for pos in range(self.n):
            self.step(pos)
        return self.end()

    def _maintenance(self, pos: int, ch: _Chunk, partial: dict) -> None:
        iteration = self.base + pos
        self._buffer(ch, iteration)
        evicted_count = ch.n
        evicted_keys = self._sorted_keys(ch) if self.events is not None else None
        last = pos == self.n - 1
        if last:
            drain = self._evict(iteration, True, max(1, self.occupancy))
            self.h_step[4:6].copy_(drain.count, non_blocking=True)
            L.Context.get().raise_pending(self.stream)
            drain.n, drain.n_dirty = (int(v) for v in self.h_step[4:6].tolist())
            self.occupancy -= drain.n
            self._buffer(drain, iteration)
            if self.chunks:
                self._flush("final", pos)
            evicted_count += drain.n
            if evicted_keys is not None:
                evicted_keys = evicted_keys + self._sorted_keys(drain)
        elif (pos + 1) % self.flush_interval == 0 and self.chunks:
            self._flush("boundary", pos)
        if self.snapshots is not None and not last:
            expect = self.snapshots.pop(pos, None)
            if expect is not None:
                used = self.cache.used.cpu().numpy().astype(bool)
                got = np.sort(self.cache.slot_key.cpu().numpy()[used])
                if not np.array_equal(expect, got):
                    raise EngineError(f"planner mirror diverged at position {pos}: "
                                      f"{len(expect)} mirrored vs {len(got)} resident")
        rec = IterationRecord(
            iteration=partial["iteration"], warmup=partial["warmup"], compute=partial["compute"],
            critical_sync=partial["critical_sync"], blocked_on_prefetch=partial["blocked_on_prefetch"],
            blocked_on_eviction=partial["blocked_on_eviction"],
            blocked_on_background=partial["blocked_on_background"], occupancy_peak=partial["occupancy_peak"],
            occupancy_end=self.occupancy, churn=partial["prefetch_count"] + evicted_count,
            prefetch_count=partial["prefetch_count"], evicted_count=evicted_count,
            critical_size=partial["critical_size"], background_size=partial["background_size"],
            lookahead=partial["lookahead"],
        )
        self.records.append(rec)
        if self.events is not None:
            self.events.append({"iteration": rec.iteration, "prefetch": partial["prefetch_keys"],
                                "ttl_updates": partial["ttl_updates"], "evicted": evicted_keys})

    def _report(self) -> RunReport:
        digest = self.store.snapshot_digest()
        totals = _totals(self.records)
        totals.update({
            "total_time": max(self.crit_end, self.bg_end, max(self.event_completes, default=0.0)),
            "peak_occupancy": self.peak_occupancy,
            "prefetched_entries": self.total_prefetched,
            "clean_evictions": self.clean_evictions,
            "dirty_evictions": self.dirty_evictions,
            "flush_count": self.flush_counter,
            "forced_flushes": self.forced_flushes,
            "store_entries_written": self.store.entries_written,
            "store_write_calls": self.store.write_calls,
        })
        return RunReport(
            kind="pipelined", config=self.cfg.to_dict(), schema=_schema_dict(self.schema), iterations_run=self.n,
            initial_lookahead=self.L0, final_lookahead=self.state.lookahead, flush_interval=self.flush_interval,
            totals=totals, metadata=dict(_METADATA), final_store_digest=digest, trace_fingerprint=self.fingerprint,
            flushes=self.flush_log, records=self.records, events=self.events, final_store=self.store,
        )


def run_pipeline(cfg: EngineConfig, schema: Schema, trace: Iterable[Batch], *, trace_fingerprint=None,
                 fault=None) -> RunReport:
    """Run the pipelined engine over a batch stream (reference run_bagpipe)."""
    batches = _materialize(trace, cfg.iterations)
    return _Pipeline(cfg, schema, batches, trace_fingerprint, fault).run()


run_bagpipe = run_pipeline


def run_synchronous_baseline(cfg: EngineConfig, schema: Schema, trace: Iterable[Batch], *,
                             trace_fingerprint=None) -> RunReport:
    """Plain fetch-train-write-back on the GPU: the bit-exact correctness oracle
    (reference engine.py:688-769).  Per batch: fetch every unique row from the
    pinned store, one fused stub-gradient + combine + SGD kernel over the rows
    in key order, write every row back."""
    batches = _materialize(trace, cfg.iterations)
    stub = cfg.stub()
    c_value, c_label, lr = f32(stub.c_value), f32(stub.c_label), f32(stub.lr)
    store = ShardedStore(schema, cfg.num_shards, cfg.seed)
    stream = torch.cuda.current_stream()
    sp = L.stream_ptr(stream)
    lib, ctx = L.lib(), L.Context.get()
    bw = cfg.sync_bandwidth
    records = []
    crit_end = 0.0
    for batch in batches:
        prep = DevicePrep.from_batch(batch, cfg.num_trainers, schema, stream=stream)
        u = prep.num_unique
        if u:
            ids = prep.tensor("d_uniq_id_s", torch.uint32, u)
            rows = store.fetch_ids_async(ids, u, stream=stream)
            store.fetch_calls += 1
            L.check(lib.bp_stub_step(ctx.handle, prep.handle, L.ptr(rows), None, None, schema.emb_dim, c_value,
                                     c_label, lr, BP_STUB_SGD, None, None, 0, None, sp), "bp_stub_step")
            store.write_ids_async(ids, rows, u, stream=stream)
            store.write_calls += 1
            store.entries_written += u
        sync = u / bw
        crit_end += cfg.fetch_latency + cfg.compute_latency + sync + cfg.fetch_latency
        records.append(IterationRecord(
            iteration=batch.iteration, warmup=False, compute=cfg.compute_latency, critical_sync=sync,
            blocked_on_prefetch=cfg.fetch_latency, blocked_on_eviction=cfg.fetch_latency,
            blocked_on_background=0.0, occupancy_peak=0, occupancy_end=0, churn=0, prefetch_count=0,
            evicted_count=0, critical_size=u, background_size=0, lookahead=0))
    ctx.raise_pending(stream)
    totals = _totals(records)
    totals.update({"total_time": crit_end, "peak_occupancy": 0, "prefetched_entries": 0, "clean_evictions": 0,
                   "dirty_evictions": 0, "flush_count": 0, "forced_flushes": 0,
                   "store_entries_written": store.entries_written, "store_write_calls": store.write_calls})
    return RunReport(kind="baseline", config=cfg.to_dict(), schema=_schema_dict(schema),
                     iterations_run=len(batches), initial_lookahead=0, final_lookahead=0, flush_interval=0,
                     totals=totals, metadata={"clock": "simulated"}, final_store_digest=store.snapshot_digest(),
                     trace_fingerprint=trace_fingerprint, records=records, events=None, final_store=store)


@dataclass
class EquivalenceResult:
    """Outcome of comparing two run digests, with an optional value-level diff."""

    equal: bool
    digest_a: str
    digest_b: str
    diffs: list = field(default_factory=list)

    def describe(self) -> str:
        if self.equal:
            return f"equal: {self.digest_a}"
        lines = [f"digest mismatch: {self.digest_a} != {self.digest_b}"]
        lines += [f"  {k.table_id}:{k.row_id} {a.tolist()} != {b.tolist()}" for k, a, b in self.diffs]
        return "\n".join(lines)


_COMPARABLE_FIELDS = ("seed", "lr", "c_value", "c_label", "num_trainers", "batch_size")


def verify_equivalence(a: RunReport, b: RunReport, diff_limit: int = 100) -> EquivalenceResult:
    """Compare final store digests of two completed runs on identical inputs."""
    if a.final_store_digest is None or b.final_store_digest is None:
        raise IncomparableRunsError("both runs must have completed")
    if a.schema != b.schema:
        raise IncomparableRunsError("runs used different schemas")
    for name in _COMPARABLE_FIELDS:
        if a.config.get(name) != b.config.get(name):
            raise IncomparableRunsError(
                f"config field {name!r} differs: {a.config.get(name)} vs {b.config.get(name)}")
    if a.iterations_run != b.iterations_run:
        raise IncomparableRunsError("runs covered different iteration counts")
    if a.trace_fingerprint is not None and b.trace_fingerprint is not None and a.trace_fingerprint != b.trace_fingerprint:
        raise IncomparableRunsError("runs used different traces")
    equal = a.final_store_digest == b.final_store_digest
    diffs = []
    if not equal and a.final_store is not None and b.final_store is not None:
        diffs = a.final_store.diff(b.final_store, limit=diff_limit)
    return EquivalenceResult(equal, a.final_store_digest, b.final_store_digest, diffs)


def fingerprint_file(path: str, batch_size: int) -> str:
    """Trace fingerprint for CLI runs: file content hash plus the batching knob."""
    h = hashlib.blake2b(digest_size=16)
    with open(path, "rb") as fh:
        while chunk := fh.read(1 << 20):
            h.update(chunk)
    return f"{h.hexdigest()}:bs={batch_size}"
