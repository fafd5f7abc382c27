"""Pipelined BagPipe engine and synchronous oracle, executed on the GPU.

API of reference engine.py:42-825 (``EngineConfig``, ``run_pipeline``,
``run_synchronous_baseline``, ``verify_equivalence``).  The control flow --
dispatch gate, forced flushes, batched round-robin write-back, simulated
clock, report -- is host arithmetic that follows reference engine.py:239-672
step for step, so reports are byte-identical.  Every per-key operation runs
on the device:

  plan emission   bp_planner_refill / bp_planner_pop        (csrc/planner.cu)
  prefetch        bp_store_fetch_lazy: zero-copy gather of written rows from
                  the pinned table, functional init of the others on the GPU
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
import os
import threading
import time
from bisect import bisect_right
from collections import deque
from dataclasses import asdict, dataclass, field
from typing import Iterable

import numpy as np
import torch

from . import _lib as L
from .device import DevicePrep, DeviceSchema, _wrap_device
from .errors import CacheCapacityError, ConfigurationError, EngineError, IncomparableRunsError
from .lookahead import auto_lookahead, planner_dump
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


class _Plan:
    """One emitted plan living in a native plan slot."""

    __slots__ = ("iteration", "lookahead", "slot", "pos", "_counts")

    def __init__(self, iteration, lookahead, slot, pos):
        self.iteration, self.lookahead, self.slot, self.pos = iteration, lookahead, slot, pos
        self._counts = None


class _Pipeline:
    EMIT_AHEAD = 3  # plans emitted ahead of dispatch (see _emit_ahead)
    PREP_AHEAD = int(os.environ.get("BAGPIPE_B200_PREP_AHEAD", "4"))  # batches prepped ahead of the window
    """One pipelined run (reference engine.py:239-649) on the native engine.

    The host keeps the reference's scalar control flow -- window refill,
    lazy pressure halving, dispatch gate, forced / boundary / final flushes,
    round-robin flusher, simulated clock, records -- and drives the native
    runtime (``csrc/engine.cu``) a few coarse calls per iteration:
    add_batch / refill / pop (planner), fetch (link stream), train (one
    synchronisation), flush (link stream).  ``begin`` / ``step(pos)`` /
    ``end`` split the reference's loop so a benchmark can time iterations.
    """

    STAGES = ("prep", "planner", "fetch", "apply", "trainer", "evict", "flush", "trainer_bwd")

    def __init__(self, cfg: EngineConfig, schema: Schema, batches: list, fingerprint, fault, device_inputs=None,
                 timing: bool = False, trainer=None, link_mode: int | None = None, threaded: bool | None = None):
        if fault not in (None, FAULT_NO_GATE, FAULT_DROP_PREFETCH):
            raise ConfigurationError(f"unknown fault {fault!r}")
        self.cfg, self.schema, self.batches = cfg, schema, batches
        self.fingerprint, self.fault = fingerprint, fault
        self.base = batches[0].iteration
        self.n = len(batches)
        self.T = cfg.num_trainers
        self.device_inputs = device_inputs  # optional {pos: (d_keys, d_labels)} already in HBM
        self.timing = bool(timing)
        self.probe = None
        self.lib = L.lib()
        self.trainer = trainer  # None: the reference's stub trainer; else e.g. dlrm.DLRMTrainer
        # iteration enqueued in _begin, counters read in _end (stub mode and
        # single-GPU DLRM): the next iteration can be enqueued in between
        self._split = trainer is None or bool(getattr(trainer, "can_split", lambda: False)())
        stub = cfg.stub()
        # Rows in the cache/store: the embedding (+ optimizer state in DLRM/Adagrad mode).
        width = trainer.row_width() if trainer is not None else schema.emb_dim
        self.row_schema = schema if width == schema.emb_dim else Schema(
            schema.num_tables, schema.rows_per_table, schema.num_dense, width)

        self.L0 = cfg.lookahead or auto_lookahead(iter(batches), cfg.cache_capacity, schema=schema)
        self.flush_interval = max(1, math.ceil(cfg.rpc_batch_proportion * self.L0))
        max_occ = max(1, max(int(b.packed_occurrences()[0].size) for b in batches))
        ec = L.EngineConfig(capacity=cfg.cache_capacity, max_occ=max_occ, seed=cfg.seed & 0xFFFFFFFFFFFFFFFF,
                            dim=width, num_ranks=self.T, c_value=f32(stub.c_value),
                            c_label=f32(stub.c_label), lr=f32(stub.lr),
                            record_keys=1 if (cfg.record_events or fault == FAULT_NO_GATE) else 0,
                            plan_slots=self.L0 + 4 + self.EMIT_AHEAD, chunk_slots=self.flush_interval + 4,
                            prep_slots=2 * self.L0 + 8 + self.EMIT_AHEAD + self.PREP_AHEAD,
                            timing=1 if timing else 0,
                            init_dims=schema.emb_dim,
                            prep_flags=2 if trainer is not None else 0)
        h = C.c_void_p()
        L.check(self.lib.bp_engine_create(L.Context.get().handle, DeviceSchema.get(self.row_schema).handle,
                                          C.byref(ec), C.byref(h)), "bp_engine_create")
        self.eng = h
        parts = L.EngineParts()
        self.lib.bp_engine_parts(h, C.byref(parts))
        self.parts = parts
        # host link: 0 = zero-copy kernels (default), 1 = copy engines + host worker pool,
        # 2 = zero-copy prefetch + copy-engine write-back with host scatter
        if link_mode is None:
            link_mode = int(os.environ.get("BAGPIPE_B200_LINK_MODE", "0"))
        L.check(self.lib.bp_engine_set_link_mode(h, link_mode, int(os.environ.get("BAGPIPE_B200_LINK_THREADS", "0"))),
                "bp_engine_set_link_mode")
        self.link_mode = link_mode
        # write-back log rows (log-structured host store; 0 = zero-copy scatter into the table)
        log_rows = int(os.environ.get("BAGPIPE_B200_LOG_ROWS", str(min(self.row_schema.total_rows, 1 << 24))))
        L.check(self.lib.bp_engine_set_write_log(h, log_rows), "bp_engine_set_write_log")
        # DLRM option: prefetches run under the dense step, not beside the EmbeddingBag
        # kernels (measured no faster on the bench step, so off by default)
        gate = int(os.environ.get("BAGPIPE_B200_LINK_GATE", "0")) if trainer is not None and self._split else 0
        L.check(self.lib.bp_engine_set_link_gate(h, gate), "bp_engine_set_link_gate")
        self.stream = torch.cuda.ExternalStream(parts.compute_stream)
        self.link = torch.cuda.ExternalStream(parts.link_stream)
        self.store = ShardedStore(self.row_schema, cfg.num_shards, cfg.seed, _handle=parts.store, _owner=self)
        self.occupancy = 0
        self.lookahead = self.L0
        self.queue: deque = deque()  # positions of the planner window
        self.source_pos = 0
        self.added: set = set()
        self.snapshots = {} if cfg.check_mirror else None
        self._adapt_pending = None
        self.free_chunks = list(range(self.flush_interval + 4))
        self.free_plans = set(range(self.L0 + 4 + self.EMIT_AHEAD))

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
        self.result = L.StepResult()
        self._inflight: dict = {}
        self.host_wait_s = 0.0  # host time blocked in bp_engine_train_end (device-bound steps)
        self._host_refs: dict = {}
        # planner thread (see _planner_loop); fault injection and event logs
        # keep the single-thread order
        # (measured: it helps device-resident batches, 0.41 -> 0.37 ms/step,
        # and slows host batches, whose uploads then contend with the
        # training thread -- so by default only with device inputs)
        # batches in pinned memory are DMA'd straight from there (no upload
        # copy on a host thread), so they take the planner thread as well
        # (compact columnar uploads: e2e 87.4-90.6M vs 84.4-88.3M
        # single-threaded over 5 runs each)
        default_threaded = bool(self.device_inputs) or (
            bool(batches) and all("pinned" in getattr(b, "_memo", {}) or "pinned_planes" in getattr(b, "_memo", {})
                                  for b in batches))
        env = os.environ.get("BAGPIPE_B200_PLANNER_THREAD")
        if env is not None:
            default_threaded = env == "1"
        self._threaded = (threaded if threaded is not None else default_threaded) and \
            fault is None and self.events is None
        self._thread = None
        self._stop = False
        self._planner_error = None
        self._cond = threading.Condition()
        self._add_lock = threading.Lock()
        self._plan_lock = threading.Lock()

    def stage_times(self) -> dict:
        """{stage: (total ms, launches)} since the last call (timing=True)."""
        ms = np.zeros(len(self.STAGES), dtype=np.float64)
        cnt = np.zeros(len(self.STAGES), dtype=np.int64)
        L.check(self.lib.bp_engine_stage_times(self.eng, ms.ctypes.data, cnt.ctypes.data), "bp_engine_stage_times")
        return {name: (float(m), int(c)) for name, m, c in zip(self.STAGES, ms, cnt)}

    def close(self) -> None:
        """Stop the planner thread and free the native engine (callers that
        step a pipeline without end())."""
        self._stop_planner()
        if getattr(self, "eng", None):
            L.check(self.lib.bp_engine_sync(self.eng), "bp_engine_sync")
            self.lib.bp_engine_destroy(self.eng)
            self.eng = None

    def __del__(self):
        try:
            if getattr(self, "eng", None):
                self.lib.bp_engine_destroy(self.eng)
                self.eng = None
        except Exception:
            pass

    # -- batches ---------------------------------------------------------------------
    def _add(self, pos: int) -> None:
        if pos in self.added:  # lock-free fast path (set membership is atomic)
            return
        with self._add_lock:  # the planner thread and the training loop may both add
            self._add_locked(pos)

    def _add_locked(self, pos: int) -> None:
        if pos in self.added:
            return
        b = self.batches[pos]
        rb = np.ascontiguousarray(b.rank_bounds(self.T), dtype=np.int64)
        dev = self.device_inputs.get(pos) if self.device_inputs else None
        packed = b._memo.get("pinned_planes") if dev is None else None
        tables = b.table_ids() if b.is_columnar else None
        if packed is not None and tables is not None and 0 < len(tables) <= 64 and \
                bool(np.all(np.diff(tables) > 0)):
            # compact columnar upload from pinned memory: row-id planes of
            # 4/2/1-byte columns + one label per example, expanded on the GPU
            buf, pl, widths = packed
            t32 = np.ascontiguousarray(tables, dtype=np.int32)
            w8 = np.ascontiguousarray(widths, dtype=np.int8)
            rc = self.lib.bp_engine_add_batch_packed(self.eng, pos, b.iteration, buf.data_ptr(), pl.data_ptr(),
                                                     b.num_examples, len(t32), t32.ctypes.data, w8.ctypes.data,
                                                     rb.ctypes.data, self.T, 1)
            L.check(rc, "bp_engine_add_batch_packed")
            self._host_refs[pos] = (buf, pl)
            self.added.add(pos)
            return
        keys, labels, _ = b.packed_occurrences()
        if dev is not None:
            kptr, lptr, on_host, n = L.ptr(dev[0]), L.ptr(dev[1]), 0, dev[0].numel()
        else:
            keys = np.ascontiguousarray(keys, dtype=np.uint64)
            labels = np.ascontiguousarray(labels, dtype=np.uint8)
            kptr, lptr, on_host, n = keys.ctypes.data, labels.ctypes.data, 1, keys.size
            # the engine copies them asynchronously: keep them alive until release
            self._host_refs[pos] = (keys, labels)
        tables = b.table_ids() if b.is_columnar else None
        if tables is not None and len(tables) and bool(np.all(np.diff(tables) > 0)):
            # Criteo layout: one key per table per example -> per-column sort
            t32 = np.ascontiguousarray(tables, dtype=np.int32)
            rc = self.lib.bp_engine_add_batch_columnar(self.eng, pos, b.iteration, kptr, lptr, b.num_examples,
                                                       len(t32), t32.ctypes.data, rb.ctypes.data, self.T, on_host)
        else:
            rc = self.lib.bp_engine_add_batch(self.eng, pos, b.iteration, kptr, lptr, n, rb.ctypes.data, self.T,
                                              on_host)
        L.check(rc, "bp_engine_add_batch")
        self.added.add(pos)

    def _release(self, pos: int) -> None:
        if pos in self.added:
            self.lib.bp_engine_release_batch(self.eng, pos)
            self.added.discard(pos)
        self._host_refs.pop(pos, None)

    # -- plan emission (reference engine.py:198-236, lookahead.py:64-123) --------
    def _plan_counts(self, plan: _Plan):
        if plan._counts is None:
            out = np.zeros(4, dtype=np.int64)
            L.check(self.lib.bp_engine_plan_counts(self.eng, plan.slot, out.ctypes.data), "bp_engine_plan_counts")
            plan._counts = out
        return plan._counts

    def _next_plan(self):
        if self._adapt_pending is not None:
            # the reference adapts lazily, when the next plan is requested
            projected = int(self._plan_counts(self._adapt_pending)[2])
            if projected > self.cfg.cache_capacity and self.lookahead > 1:
                self.lookahead = max(1, self.lookahead // 2)
            self._adapt_pending = None
        while len(self.queue) < self.lookahead and self.source_pos < self.n:
            pos = self.source_pos
            self.source_pos += 1
            self._add(pos)
            L.check(self.lib.bp_engine_refill(self.eng, pos), "bp_engine_refill")
            self.queue.append(pos)
        if not self.queue:
            return None
        pos = self.queue.popleft()
        slot = C.c_int32()
        L.check(self.lib.bp_engine_pop(self.eng, pos, C.byref(slot)), "bp_engine_pop")
        with self._plan_lock:
            if slot.value not in self.free_plans:
                raise EngineError("plan ring overrun")
            self.free_plans.discard(slot.value)
        plan = _Plan(self.batches[pos].iteration, self.lookahead, slot.value, pos)
        self._adapt_pending = plan
        if self.snapshots is not None:
            self._plan_counts(plan)  # the pop ran on the plan stream: wait for it before dumping
            keys, _, flags = planner_dump(self.parts.planner, self.stream)
            self.snapshots[pos] = np.sort(keys[(flags & 2) != 0])
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
        L.check(self.lib.bp_engine_fetch(self.eng, plan.slot), "bp_engine_fetch")
        self.staged[plan.iteration - self.base] = (plan, arrival)

    def _dispatch_until(self, cur: int) -> None:
        if self._thread is not None:
            return self._dispatch_until_threaded(cur)
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

    # -- write-back (reference engine.py:350-377) ---------------------------------
    def _flush(self, kind: str, pos: int) -> None:
        flusher = self.flush_counter % self.T
        count = 0
        if self.chunks:
            slots = np.asarray([c[0] for c in self.chunks], dtype=np.int32)
            L.check(self.lib.bp_engine_flush(self.eng, slots.ctypes.data, len(slots)), "bp_engine_flush")
            count = self._merged_count()
            self.free_chunks.extend(int(s) for s in slots)
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
            return sum(c[2] for c in self.chunks)
        keys = [k[d] for k, d in (self._chunk_keys(c[0], c[1], with_dirty=True) for c in self.chunks)]
        return int(np.unique(np.concatenate(keys)).size)

    def _chunk_keys(self, slot: int, n: int, with_dirty: bool = False):
        keys = np.zeros(n, dtype=np.uint64)
        L.check(self.lib.bp_engine_chunk_keys(self.eng, slot, keys.ctypes.data, n), "bp_engine_chunk_keys")
        if not with_dirty:
            return keys
        view = L.EvictBuffers()
        self.lib.bp_engine_chunk_view(self.eng, slot, C.byref(view))
        dirty = L.to_host(_wrap_device(view.d_dirty, torch.uint8, max(n, 1)), n).astype(bool)
        return keys, dirty

    def _buffer(self, slot: int, n: int, n_dirty: int, iteration: int) -> None:
        self.clean_evictions += n - n_dirty
        self.dirty_evictions += n_dirty
        if n_dirty:
            self.chunks.append((slot, n, n_dirty))
            if self.min_unflushed_ttl is None or iteration < self.min_unflushed_ttl:
                self.min_unflushed_ttl = iteration
        else:
            self.free_chunks.append(slot)

    def _take_chunk(self) -> int:
        if not self.free_chunks:
            raise EngineError("eviction chunk ring overrun")
        return self.free_chunks.pop(0)

    # -- per iteration ---------------------------------------------------------------
    def _dispatch_until_threaded(self, cur: int) -> None:
        while True:
            with self._cond:
                while not self.pending and not self.exhausted:
                    self._cond.wait()
                if self._planner_error is not None:
                    raise self._planner_error
                if not self.pending:
                    return
                plan = self.pending[0]
                if self._dispatch_pos(plan) > cur:
                    return
                self.pending.popleft()
                self._cond.notify_all()
            self._dispatch(plan, cur)

    def _planner_loop(self) -> None:
        """Planner thread: batch preps and plan emission (the reference's
        emit_next_plan + lazy adapt, in order) run here, ahead of the
        training loop, whose thread keeps only dispatch, training and
        write-back.  ctypes drops the GIL inside every native call, so the
        two threads' CUDA API calls overlap."""
        try:
            torch.cuda.set_device(self._device)  # the CUDA current device is per thread
            while True:
                with self._cond:
                    while not self._stop and (self.exhausted or len(self.pending) >= self.EMIT_AHEAD):
                        self._cond.wait()
                    if self._stop:
                        return
                for p in range(self.source_pos, min(self.n, self.source_pos + self.PREP_AHEAD)):
                    self._add(p)
                plan = self._next_plan()
                with self._cond:
                    if plan is None:
                        self.exhausted = True
                    else:
                        self.pending.append(plan)
                    self._cond.notify_all()
        except BaseException as err:  # surfaced on the training thread
            with self._cond:
                self._planner_error = err
                self.exhausted = True
                self._cond.notify_all()

    def _stop_planner(self) -> None:
        if self._thread is not None:
            with self._cond:
                self._stop = True
                self._cond.notify_all()
            self._thread.join()
            self._thread = None

    def begin(self) -> None:
        self._wall0 = time.perf_counter()
        self.host_wait_s = 0.0
        self._wall_marks = []
        if self._threaded:
            self._device = torch.cuda.current_device()
            self._thread = threading.Thread(target=self._planner_loop, name="bagpipe-planner", daemon=True)
            self._thread.start()
        self._dispatch_until(-1)

    def step(self, pos: int, early: bool = True) -> None:
        """One reference iteration.  In stub mode the next iteration is
        enqueued on the GPU before this one's counters are read (when its plan
        is already staged), so host bookkeeping overlaps device work; the
        reference order of every host decision is unchanged."""
        if pos > 0:
            self._dispatch_until(pos - 1)
        if pos not in self._inflight:
            self._begin(pos)
        nxt = pos + 1
        if (early and self._split and self.fault is None and self.events is None and self.snapshots is None
                and nxt < self.n and nxt in self.staged and nxt not in self._inflight
                and len(self.free_chunks) >= (2 if nxt == self.n - 1 else 1)):
            self._begin(nxt)
        if self._split and self._thread is None:
            # plan emission (planner stream) overlaps the queued GPU work
            self._emit_ahead()
        self._end(pos)

    def _begin(self, pos: int) -> None:
        lib = self.lib
        batch = self.batches[pos]
        iteration = batch.iteration
        staged = self.staged.pop(pos, None)
        if staged is None:
            raise EngineError(f"no staged prefetch for position {pos}")
        plan, arrival = staged
        if plan.iteration != iteration:
            raise EngineError(f"plan {plan.iteration} misaligned with batch {iteration}")
        skip_key, has_skip = 0, 0
        if self.fault == FAULT_DROP_PREFETCH and not self.drop_done and pos >= self.n // 2 \
                and self._plan_counts(plan)[0]:
            # Drop the first (smallest) prefetched key: it is neither inserted
            # nor TTL-updated, so the lookup must miss (reference engine.py:512-523).
            skip_key = int(self._plan_keys(plan, 1)[0])
            has_skip = 1
            self.drop_done = True
        last = pos == self.n - 1
        nxt = pos + 1 if pos + 1 < self.n else -1
        if nxt >= 0:
            self._add(nxt)
        chunk = self._take_chunk()
        drain = self._take_chunk() if last else -1
        self._inflight[pos] = (plan, arrival, skip_key, has_skip, nxt, chunk, drain)
        if self.trainer is None:
            L.check(lib.bp_engine_train_begin(self.eng, pos, plan.slot, nxt, skip_key, has_skip, chunk, drain),
                    "bp_engine_train_begin")
        elif self._split:
            self.trainer.train_begin(self, pos, plan, nxt, skip_key, has_skip, chunk, drain)

    def _end(self, pos: int) -> None:
        cfg, lib = self.cfg, self.lib
        bw = cfg.sync_bandwidth
        iteration = self.batches[pos].iteration
        plan, arrival, skip_key, has_skip, nxt, chunk, drain = self._inflight.pop(pos)
        res = self.result
        if self._split:
            t0 = time.perf_counter()
            L.check(lib.bp_engine_train_end(self.eng, C.byref(res)), "bp_engine_train_end")
            self.host_wait_s += time.perf_counter() - t0  # host blocked on the device
        else:
            self.trainer.train(self, pos, plan, nxt, skip_key, has_skip, chunk, drain, res)
        if res.err.code:
            L.raise_error_record(res.err)
        with self._plan_lock:
            self.free_plans.add(plan.slot)
        u, n_ins, crit_count = int(res.unique), int(res.inserted), int(res.critical)
        n_ev, n_ev_dirty = int(res.evicted), int(res.evicted_dirty)
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
            critical_size = crit_count if nxt >= 0 else 0
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
            ttl = self._plan_ttls(plan)
            pf = unpack_keys(self._plan_keys(plan, int(self._plan_counts(plan)[0])))
            if has_skip:
                lost = unpack_key(skip_key)
                ttl = [(k, t) for k, t in ttl if k != lost]
                pf = pf[1:]
            partial["prefetch_keys"] = pf
            partial["ttl_updates"] = ttl
        self._maintenance(pos, chunk, n_ev, n_ev_dirty, drain, int(res.drained), int(res.drained_dirty), partial)
        self._release(pos)
        if self._thread is None:
            self._emit_ahead()

    def _emit_ahead(self) -> None:
        """Emit plans ahead of their dispatch while the previous pop already
        finished on the device (non-blocking query), so the reference's lazy
        adapt (which needs the previous plan's projected occupancy) never
        stalls the host on a pop it has just queued.  The plan sequence is a
        function of the trace and capacity only, so emitting earlier does
        not change any plan.  Batch preps run PREP_AHEAD batches ahead of
        the window on their own stream, so an emission only waits for the
        planner's refill + pop."""
        for p in range(self.source_pos, min(self.n, self.source_pos + self.PREP_AHEAD)):
            self._add(p)
        while len(self.pending) < self.EMIT_AHEAD and not self.exhausted:
            prev = self._adapt_pending
            if prev is not None:
                ready = C.c_int32()
                L.check(self.lib.bp_engine_plan_ready(self.eng, prev.slot, C.byref(ready)), "bp_engine_plan_ready")
                if not ready.value:
                    return
            plan = self._next_plan()
            if plan is None:
                self.exhausted = True
                return
            self.pending.append(plan)

    def _plan_keys(self, plan, n: int) -> np.ndarray:
        view = L.PlanBuffers()
        self.lib.bp_engine_plan_view(self.eng, plan.slot, C.byref(view), None)
        return L.to_host(_wrap_device(view.d_prefetch_keys, torch.uint64, max(n, 1)), n)

    def _plan_ttls(self, plan) -> list:
        prep = C.c_void_p()
        L.check(self.lib.bp_engine_prep(self.eng, plan.pos, C.byref(prep)), "bp_engine_prep")
        pv = L.PrepView()
        self.lib.bp_prep_get_view(prep, C.byref(pv))
        u = int(L.to_host(_wrap_device(pv.d_num_unique, torch.int64, 1))[0])
        view = L.PlanBuffers()
        self.lib.bp_engine_plan_view(self.eng, plan.slot, C.byref(view), None)
        keys = unpack_keys(L.to_host(_wrap_device(pv.d_uniq_key_k, torch.uint64, max(u, 1)), u))
        ttls = L.to_host(_wrap_device(view.d_ttl_k, torch.int64, max(u, 1)), u).tolist()
        return list(zip(keys, ttls))

    def end(self) -> RunReport:
        self._stop_planner()
        if self._planner_error is not None:
            raise self._planner_error
        if not self.exhausted and (self.pending or self._next_plan() is not None):
            raise EngineError("planner emitted more plans than batches")
        L.check(self.lib.bp_engine_sync(self.eng), "bp_engine_sync")
        return self._report()

    def run(self) -> RunReport:
        try:
            self.begin()
            for pos in range(self.n):
                self.step(pos)
            return self.end()
        finally:
            self._stop_planner()  # also on errors: the thread holds the pipeline alive

    def _maintenance(self, pos, chunk, n_ev, n_ev_dirty, drain, n_dr, n_dr_dirty, partial) -> None:
        iteration = self.base + pos
        evicted_keys = None
        if self.events is not None:
            evicted_keys = unpack_keys(np.sort(self._chunk_keys(chunk, n_ev)))
        self._buffer(chunk, n_ev, n_ev_dirty, iteration)
        evicted_count = n_ev
        last = pos == self.n - 1
        if last:
            self.occupancy -= n_dr
            if evicted_keys is not None:
                evicted_keys = evicted_keys + unpack_keys(np.sort(self._chunk_keys(drain, n_dr)))
            self._buffer(drain, n_dr, n_dr_dirty, iteration)
            if self.chunks:
                self._flush("final", pos)
            evicted_count += n_dr
        elif (pos + 1) % self.flush_interval == 0 and self.chunks:
            self._flush("boundary", pos)
        if self.snapshots is not None and not last:
            expect = self.snapshots.pop(pos, None)
            if expect is not None:
                view = L.CacheView()
                self.lib.bp_cache_get_view(self.parts.cache, C.byref(view))
                used = L.to_host(_wrap_device(view.d_used, torch.uint8, view.capacity)).astype(bool)
                got = np.sort(L.to_host(_wrap_device(view.d_slot_key, torch.uint64, view.capacity))[used])
                if not np.array_equal(expect, got):
                    raise EngineError(f"planner mirror diverged at position {pos}: "
                                      f"{len(expect)} mirrored vs {len(got)} resident")
        if getattr(self, "_wall_marks", None) is not None:
            self._wall_marks.append(time.perf_counter())
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
        marks = getattr(self, "_wall_marks", None) or []
        t0 = getattr(self, "_wall0", None)
        wall = [round((b - a) * 1e3, 6) for a, b in zip([t0] + marks[:-1], marks)] if t0 is not None else []
        measured = {"clock": "measured (host perf_counter; device stage spans when the engine times stages)",
                    "wall_ms_per_iteration": wall, "wall_ms_total": round(sum(wall), 6),
                    "device": torch.cuda.get_device_name() if torch.cuda.is_available() else None}
        if self.timing:
            measured["stage_ms"] = {k: v[0] for k, v in self.stage_times().items()}
        return RunReport(
            kind="pipelined", config=self.cfg.to_dict(), schema=_schema_dict(self.schema), iterations_run=self.n,
            initial_lookahead=self.L0, final_lookahead=self.lookahead, flush_interval=self.flush_interval,
            totals=totals, metadata=dict(_METADATA), final_store_digest=digest, trace_fingerprint=self.fingerprint,
            flushes=self.flush_log, records=self.records, events=self.events, final_store=self.store,
            measured=measured,
        )


def run_pipeline(cfg: EngineConfig, schema: Schema, trace: Iterable[Batch], *, trace_fingerprint=None,
                 fault=None, measure_stages: bool = False, device_inputs=None) -> RunReport:
    """Run the pipelined engine over a batch stream (reference run_bagpipe).
    measure_stages: also record per-stage device time (CUDA events) into the
    report's measured-timing sidecar; device_inputs: {position: (d_keys,
    d_labels)} of batches already in HBM (ingest.DeviceTrace.batch_inputs)."""
    batches = _materialize(trace, cfg.iterations)
    return _Pipeline(cfg, schema, batches, trace_fingerprint, fault, timing=measure_stages,
                     device_inputs=device_inputs).run()


run_bagpipe = run_pipeline


def run_dlrm(cfg: EngineConfig, schema: Schema, trace: Iterable[Batch], dlrm_cfg=None, *, trace_fingerprint=None,
             model=None, exchange=None):
    """Pipelined BagPipe training of a DLRM (dense MLPs in PyTorch, embedding
    path native).  Returns (RunReport, DLRMTrainer); batches need dense
    features (``Batch.dense``).  N > 1: pass this rank's table-sharded batches
    (shard.shard_batches) and a hybrid.EmbeddingExchange."""
    from .dlrm import DLRMConfig, DLRMTrainer

    batches = _materialize(trace, cfg.iterations)
    dcfg = dlrm_cfg or DLRMConfig(emb_lr=cfg.lr, mlp_lr=cfg.lr)
    trainer = DLRMTrainer(dcfg, schema.num_dense, schema.num_tables, schema.emb_dim, model=model, exchange=exchange)
    pipe = _Pipeline(cfg, schema, batches, trace_fingerprint, None, trainer=trainer)
    report = pipe.run()
    return report, trainer


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
            rows = store.fetch_ids_async(ids, u, stream=stream, d_keys=prep.tensor("d_uniq_key_s", torch.uint64, u))
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
