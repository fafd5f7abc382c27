"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY, never part of the product path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg import this module, and only as the checker or as the
timed CPU baseline.  The product (paper_2202_12429_b200) never imports it.

A numpy restatement of the reference (embcache 0.1.0, /root/reference/pkg)
algorithm for the embedding-access path, written as whole-batch vector
operations over dense per-key arrays instead of the reference's per-key
dictionary loops:

  hashing / init     reference hashing.py:42-79, store.py:29-42
  unique keys        reference traces.py:91-103, engine.py:142-182
  Algorithm 1        reference lookahead.py:64-123 (refill / pop / halving)
  cache contents     reference cache.py:99-286 (insert / TTL / update /
                     evict / drain, content_checksum, canonical_digest)
  stub trainer       reference trainer.py:37-53, 92-105, 140-146
  baseline engine    reference engine.py:688-769
  pipeline data path reference engine.py:302-452 (gate, forced flush,
                     cadence, TTL cache, dirty write-back); the simulated
                     clock and report layout are pinned separately by the
                     golden reports the reference itself produced.

Parity is PINNED: tests/test_oracle.py checks this module against the golden
vectors of tests/golden/ (generated from the reference by
tests/golden/make_golden.py): published hash vectors, the worked-example and
small-fixture plan streams, Criteo-Kaggle plan digests, and final store
digests (f2c6d9f7... for the acceptance fixture).
"""

from __future__ import annotations

import hashlib
import math

import numpy as np

FNV_OFFSET = np.uint64(0xCBF29CE484222325)
FNV_PRIME = np.uint64(0x100000001B3)
SHIFT = np.uint64(44)
ROWMASK = np.uint64((1 << 44) - 1)


# ------------------------------------------------------------------ hashing
def fnv_cols(*cols) -> np.ndarray:
    """FNV-1a 64 over the little-endian bytes of each u64 column (hashing.py:42-51)."""
    h = np.full(np.shape(cols[0]), FNV_OFFSET, dtype=np.uint64)
    for c in cols:
        c = np.asarray(c, dtype=np.uint64)
        for s in range(8):
            h = (h ^ ((c >> np.uint64(8 * s)) & np.uint64(255))) * FNV_PRIME
    return h


def splitmix(x) -> np.ndarray:
    """splitmix64 finaliser of x + gamma (hashing.py:62-67)."""
    z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def init_rows(seed: int, tables, rows, dim: int) -> np.ndarray:
    """Functional initial values (store.py:29-42): f64 math, one f32 rounding."""
    t = np.asarray(tables, dtype=np.uint64)
    r = np.asarray(rows, dtype=np.uint64)
    n = t.size
    j = np.arange(dim, dtype=np.uint64)
    h = fnv_cols(np.repeat(t, dim), np.repeat(r, dim), np.tile(j, n))
    m = splitmix(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ h)
    unit = (m >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return (-0.05 + 0.1 * unit).astype(np.float32).reshape(n, dim)


# ------------------------------------------------------------ batch layout
def pack(tables, rows) -> np.ndarray:
    return (np.asarray(tables, dtype=np.uint64) << SHIFT) | np.asarray(rows, dtype=np.uint64)


def batch_occurrences(batch):
    """(packed keys, labels, example offsets) in occurrence order."""
    if getattr(batch, "rows", None) is not None and getattr(batch, "_examples", None) is None:
        n, nt = batch.rows.shape
        tids = getattr(batch, "tables", None)
        keys = pack((np.arange(nt) if tids is None else tids)[None, :], batch.rows).reshape(-1)
        return keys, np.repeat(np.asarray(batch.labels, dtype=np.float32), nt), np.arange(n + 1) * nt
    keys, labels, offs = [], [], [0]
    for ex in batch.examples:
        for k in ex.sparse:
            keys.append((int(k[0]) << 44) | int(k[1]))
            labels.append(ex.label)
        offs.append(len(keys))
    return np.asarray(keys, dtype=np.uint64), np.asarray(labels, dtype=np.float32), np.asarray(offs)


def first_order_unique(keys: np.ndarray):
    """Unique keys in first-occurrence order and each occurrence's index into them."""
    if keys.size == 0:
        return keys, np.zeros(0, dtype=np.int64)
    sorted_u, first, inv = np.unique(keys, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")           # sorted index -> first-occurrence rank
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    return sorted_u[order], rank[inv]


# ----------------------------------------------------------- cache contents
def content_checksum(keys, ttl, dirty, values) -> int:
    """XOR over entries of a splitmix chain over (t<<44 ^ r), ttl, dirty<<63
    and every f32 word of the value (cache.py:249-272); order-independent."""
    keys = np.asarray(keys, dtype=np.uint64)
    if keys.size == 0:
        return 0
    word = splitmix(keys)
    word = splitmix(word ^ np.asarray(ttl, dtype=np.int64).astype(np.uint64))
    word = splitmix(word ^ (np.asarray(dirty, dtype=np.uint64) << np.uint64(63)))
    vals = np.ascontiguousarray(values, dtype=np.float32).view(np.uint32).astype(np.uint64)
    for j in range(vals.shape[1]):
        word = splitmix(word ^ vals[:, j])
    return int(np.bitwise_xor.reduce(word))


def canonical_digest(keys, ttl, dirty, values) -> str:
    """blake2b-128 over key-sorted records <i8 table, row, ttl, dirty> + <f4
    value (cache.py:274-286); one update over the concatenated records equals
    the reference's per-entry updates."""
    keys = np.asarray(keys, dtype=np.uint64)
    order = np.argsort(keys, kind="stable")
    k = keys[order]
    dim = np.shape(values)[1] if np.ndim(values) == 2 else 0
    rec = np.zeros(k.size, dtype=[("h", "<i8", (4,)), ("v", "<f4", (dim,))])
    rec["h"][:, 0] = (k >> SHIFT).astype(np.int64)
    rec["h"][:, 1] = (k & ROWMASK).astype(np.int64)
    rec["h"][:, 2] = np.asarray(ttl, dtype=np.int64)[order]
    rec["h"][:, 3] = np.asarray(dirty, dtype=np.int64)[order]
    if k.size:
        rec["v"] = np.asarray(values, dtype=np.float32)[order]
    h = hashlib.blake2b(digest_size=16)
    h.update(rec.tobytes())
    return h.hexdigest()


class DictCache:
    """The reference DynamicCache's contents as a dict key -> [value, ttl,
    dirty] (cache.py:99-247): enough to replay an API scenario and checksum
    it; capacity/ordering errors are exercised on the GPU object itself."""

    def __init__(self):
        self.ent = {}

    def prefetch(self, keys, values, ttls):
        for k, v, t in zip(keys, values, ttls):
            assert k not in self.ent
            self.ent[int(k)] = [np.asarray(v, dtype=np.float32).copy(), int(t), False]

    def set_ttl(self, keys, ttls):
        for k, t in zip(keys, ttls):
            self.ent[int(k)][1] = int(t)

    def update(self, keys, values, mask):
        for k, v, m in zip(keys, values, mask):
            e = self.ent[int(k)]
            e[0] = np.asarray(v, dtype=np.float32).copy()
            e[2] = e[2] or bool(m)

    def release(self, pred):
        gone = sorted(k for k, e in self.ent.items() if pred(e))
        out = [(k, self.ent[k][0], self.ent[k][2]) for k in gone]
        for k in gone:
            del self.ent[k]
        return out

    def arrays(self):
        ks = sorted(self.ent)
        dim = len(next(iter(self.ent.values()))[0]) if ks else 0
        vals = np.asarray([self.ent[k][0] for k in ks], dtype=np.float32).reshape(len(ks), dim)
        return (np.asarray(ks, dtype=np.uint64), np.asarray([self.ent[k][1] for k in ks], dtype=np.int64),
                np.asarray([self.ent[k][2] for k in ks], dtype=bool), vals)

    def checksum(self) -> int:
        return content_checksum(*self.arrays())

    def digest(self) -> str:
        return canonical_digest(*self.arrays())


def shard_of(tables, rows, num_shards: int) -> np.ndarray:
    """fnv1a64(t, r) mod num_shards (store.py:80-88, 100-104)."""
    return (fnv_cols(tables, rows) % np.uint64(num_shards)).astype(np.int64)


# ------------------------------------------------------------- Algorithm 1
class Planner:
    """Streaming Algorithm 1 over dense key ids.

    tracker[id] = last iteration of the key inside the window (-1: absent);
    mirror[id]  = the planner's copy of the cache contents.
    """

    def __init__(self, lookahead: int, capacity: int):
        self.lookahead = lookahead
        self.capacity = capacity
        self.ids: dict = {}
        self.last = np.full(1024, -1, dtype=np.int64)
        self.tracked = np.zeros(1024, dtype=bool)
        self.mirror = np.zeros(1024, dtype=bool)
        self.queue: list = []
        self.n_tracked = 0
        self.projected = 0
        self.insertions = self.removals = self.peak_occupancy = self.peak_projected = 0

    def _id(self, keys: np.ndarray) -> np.ndarray:
        out = np.empty(keys.size, dtype=np.int64)
        for i, k in enumerate(keys.tolist()):
            out[i] = self.ids.setdefault(k, len(self.ids))
        if len(self.ids) > self.last.size:
            grow = max(len(self.ids), 2 * self.last.size)
            self.last = np.concatenate([self.last, np.full(grow - self.last.size, -1, dtype=np.int64)])
            self.tracked = np.concatenate([self.tracked, np.zeros(grow - self.tracked.size, dtype=bool)])
            self.mirror = np.concatenate([self.mirror, np.zeros(grow - self.mirror.size, dtype=bool)])
        return out

    def push(self, iteration: int, uniq: np.ndarray) -> None:
        ids = self._id(uniq)
        self.n_tracked += int((~self.tracked[ids]).sum())
        self.tracked[ids] = True
        self.last[ids] = iteration
        self.queue.append((iteration, uniq, ids))

    def emit(self, source):
        """One emission: refill to L, pop front.  Returns (iteration, prefetch
        sorted, uniq (first order), ttl, evict sorted, lookahead) or None."""
        while len(self.queue) < self.lookahead:
            nxt = next(source, None)
            if nxt is None:
                break
            self.push(*nxt)
        self.projected = self.n_tracked
        self.peak_projected = max(self.peak_projected, self.projected)
        if not self.queue:
            return None
        iteration, uniq, ids = self.queue.pop(0)
        ttl = self.last[ids]
        pf = ~self.mirror[ids]
        ev = ttl == iteration
        resident_before = int(self.mirror.sum())
        self.mirror[ids] = True
        self.mirror[ids[ev]] = False
        self.tracked[ids[ev]] = False
        self.n_tracked -= int(ev.sum())
        self.insertions += int(pf.sum())
        self.removals += int(ev.sum())
        self.peak_occupancy = max(self.peak_occupancy, resident_before + int(pf.sum()))
        return iteration, np.sort(uniq[pf]), uniq, ttl.copy(), np.sort(uniq[ev]), self.lookahead

    def adapt(self) -> bool:
        if self.projected > self.capacity and self.lookahead > 1:
            self.lookahead = max(1, self.lookahead // 2)
            return True
        return False


def plan_stream(batches, lookahead: int, capacity: int):
    """All plans of a trace (plan_trace) plus final planner statistics."""
    pl = Planner(lookahead, capacity)
    src = ((b.iteration, first_order_unique(batch_occurrences(b)[0])[0]) for b in batches)
    plans = []
    while (p := pl.emit(src)) is not None:
        plans.append(p)
        pl.adapt()
    stats = dict(lookahead=pl.lookahead, insertions=pl.insertions, removals=pl.removals,
                 peak_occupancy=pl.peak_occupancy, peak_projected=pl.peak_projected)
    return plans, stats


def auto_lookahead(batches, capacity: int) -> int:
    seen: set = set()
    n = 0
    for b in batches:
        seen.update(np.unique(batch_occurrences(b)[0]).tolist())
        if len(seen) > capacity:
            if n == 0:
                raise ValueError("first batch alone exceeds capacity")
            return n
        n += 1
    if n == 0:
        raise ValueError("empty prefix")
    return n


# ------------------------------------------------------------ stub trainer
def batch_gradients(batch, values: np.ndarray, num_trainers: int, c_value: float, c_label: float):
    """Combined stub gradient per batch-unique key (first-occurrence order).

    Per rank r (contiguous examples [r*n/T, (r+1)*n/T)): np.add.at in
    occurrence order from +0.0; ranks combined in ascending order.  Keys absent
    from a rank contribute an exact +0.0 (x + 0.0 == x for every x reachable
    here), which equals skipping them as the reference does.
    """
    keys, labels, offs = batch_occurrences(batch)
    uniq, inv = first_order_unique(keys)
    scaled = np.float32(c_value) * values
    bias = (np.float32(c_label) * (labels - np.float32(0.5)))[:, None]
    occ = scaled[inv] + bias
    n = len(offs) - 1
    combined = np.zeros_like(values)
    for r in range(num_trainers):
        lo, hi = offs[r * n // num_trainers], offs[(r + 1) * n // num_trainers]
        g = np.zeros_like(values)
        np.add.at(g, inv[lo:hi], occ[lo:hi])
        combined = combined + g
    return uniq, combined


def sgd(values: np.ndarray, grads: np.ndarray, lr: float) -> np.ndarray:
    return values - np.float32(lr) * grads


# --------------------------------------------------------------------- store
class Store:
    """Dense lazily-initialised table (written rows kept, others functional)."""

    def __init__(self, rows_per_table, dim: int, seed: int):
        self.rows_per_table = tuple(rows_per_table)
        self.base = np.concatenate([[0], np.cumsum(self.rows_per_table)]).astype(np.int64)
        self.dim, self.seed = dim, seed
        self.values: dict = {}

    def fetch(self, keys: np.ndarray) -> np.ndarray:
        out = init_rows(self.seed, keys >> SHIFT, keys & ROWMASK, self.dim)
        for i, k in enumerate(keys.tolist()):
            v = self.values.get(k)
            if v is not None:
                out[i] = v
        return out

    def write(self, keys: np.ndarray, rows: np.ndarray) -> None:
        for k, v in zip(keys.tolist(), rows):
            self.values[k] = v.copy()

    def digest(self) -> str:
        h = hashlib.blake2b(digest_size=16)
        by_table: dict = {}
        for k, v in self.values.items():
            by_table.setdefault(k >> 44, []).append((k & ((1 << 44) - 1), v))
        for t, rows in enumerate(self.rows_per_table):
            for lo in range(0, rows, 1 << 20):
                hi = min(rows, lo + (1 << 20))
                mat = init_rows(self.seed, np.full(hi - lo, t), np.arange(lo, hi), self.dim)
                for r, v in by_table.get(t, []):
                    if lo <= r < hi:
                        mat[r - lo] = v
                h.update(mat.astype("<f4").tobytes())
        return h.hexdigest()


def baseline(batches, rows_per_table, dim: int, seed: int, num_trainers: int, lr=0.01, c_value=0.01,
             c_label=0.001) -> Store:
    """Synchronous fetch -> grad -> combine -> SGD -> write-back (engine.py:688-769)."""
    store = Store(rows_per_table, dim, seed)
    for b in batches:
        keys, _, _ = batch_occurrences(b)
        uniq, _ = first_order_unique(keys)
        vals = store.fetch(uniq)
        _, g = batch_gradients(b, vals, num_trainers, c_value, c_label)
        store.write(uniq, sgd(vals, g, lr))
    return store


# ------------------------------------------------------ pipeline data path
class OraclePipeline:
    """The pipelined engine's data path (engine.py:302-452) without the clock.

    Dispatch position of plan x: min(first flush boundary >= x - L_x, x - 1)
    (-1 before iteration 0); forced flush when an unflushed dirty eviction has
    ttl <= x - L_x; flush on (pos+1) % interval == 0; final drain + flush.
    ``step(pos)`` runs one iteration; ``stats`` collects per-iteration counters.
    """

    def __init__(self, batches, rows_per_table, dim: int, seed: int, num_trainers: int, capacity: int,
                 lookahead: int, rpc: float, lr=0.01, c_value=0.01, c_label=0.001):
        self.batches, self.dim, self.T = batches, dim, num_trainers
        self.capacity, self.lr, self.c_value, self.c_label = capacity, lr, c_value, c_label
        self.base = batches[0].iteration
        self.n = len(batches)
        self.L0 = lookahead or auto_lookahead(batches, capacity)
        self.interval = max(1, math.ceil(rpc * self.L0))
        self.store = Store(rows_per_table, dim, seed)
        self.planner = Planner(self.L0, capacity)
        self.src = ((b.iteration, first_order_unique(batch_occurrences(b)[0])[0]) for b in batches)
        self.cache: dict = {}  # key -> [row f32[dim], ttl, dirty]
        self.pending, self.staged, self.buffered = [], {}, []
        self.exhausted = False
        self.min_unflushed = None
        self.stats: list = []

    def _dispatch_pos(self, plan) -> int:
        pos = plan[0] - self.base
        s = pos - plan[5]
        if s < 0:
            return -1
        p = self.interval
        return min(((s + p) // p) * p - 1, pos - 1)

    def _flush(self) -> None:
        merged: dict = {}
        for keys, rows in self.buffered:
            for k, v in zip(keys, rows):
                merged[k] = v
        if merged:
            ks = np.asarray(sorted(merged), dtype=np.uint64)
            self.store.write(ks, np.stack([merged[k] for k in ks.tolist()]))
        self.buffered.clear()
        self.min_unflushed = None

    def _dispatch_until(self, cur: int) -> None:
        while True:
            if not self.pending:
                if self.exhausted:
                    return
                plan = self.planner.emit(self.src)
                if plan is None:
                    self.exhausted = True
                    return
                self.planner.adapt()
                self.pending.append(plan)
            plan = self.pending[0]
            if self._dispatch_pos(plan) > cur:
                return
            self.pending.pop(0)
            if self.min_unflushed is not None and self.min_unflushed <= plan[0] - plan[5]:
                self._flush()
            self.staged[plan[0] - self.base] = (plan, self.store.fetch(plan[1]))

    def _evict(self, pred):
        gone = sorted(k for k, e in self.cache.items() if pred(e))
        return gone, [self.cache.pop(k) for k in gone]

    def _buffer(self, gone, ent, iteration) -> int:
        dirty = [(k, e[0]) for k, e in zip(gone, ent) if e[2]]
        if dirty:
            self.buffered.append(([k for k, _ in dirty], [v for _, v in dirty]))
            if self.min_unflushed is None:
                self.min_unflushed = iteration
        return len(dirty)

    def begin(self) -> None:
        self._dispatch_until(-1)

    def step(self, pos: int) -> None:
        cache = self.cache
        if pos > 0:
            self._dispatch_until(pos - 1)
        (iteration, pf, uniq, ttl, _, _), pf_rows = self.staged.pop(pos)
        ttl_of = dict(zip(uniq.tolist(), ttl.tolist()))
        if len(cache) + len(pf) > self.capacity:
            raise RuntimeError(f"capacity exceeded at {iteration}")
        for k, v in zip(pf.tolist(), pf_rows):
            cache[k] = [v.copy(), ttl_of[k], False]
        for k, t in ttl_of.items():
            cache[k][1] = t
        occ_peak = len(cache)
        keys = uniq.tolist()
        vals = np.stack([cache[k][0] for k in keys]) if keys else np.zeros((0, self.dim), np.float32)
        _, g = batch_gradients(self.batches[pos], vals, self.T, self.c_value, self.c_label)
        new = sgd(vals, g, self.lr)
        dirty = (g != 0).any(axis=1)
        for i, k in enumerate(keys):
            e = cache[k]
            e[0] = new[i]
            e[2] = e[2] or bool(dirty[i])
        gone, ent = self._evict(lambda e: e[1] <= iteration)
        n_dirty = self._buffer(gone, ent, iteration)
        if pos == self.n - 1:
            gone2, ent2 = self._evict(lambda e: True)
            self._buffer(gone2, ent2, iteration)
            self._flush()
            gone = gone + gone2
        elif (pos + 1) % self.interval == 0 and self.buffered:
            self._flush()
        self.stats.append({"prefetch": len(pf), "evicted": len(gone), "dirty": n_dirty, "occupancy_peak": occ_peak,
                           "occupancy_end": len(cache), "unique": len(keys)})


def pipeline(batches, rows_per_table, dim: int, seed: int, num_trainers: int, capacity: int, lookahead: int,
             rpc: float, lr=0.01, c_value=0.01, c_label=0.001):
    """Run the whole pipeline data path; returns (store, per-iteration counters)."""
    run = OraclePipeline(batches, rows_per_table, dim, seed, num_trainers, capacity, lookahead, rpc, lr, c_value,
                         c_label)
    run.begin()
    for pos in range(run.n):
        run.step(pos)
    return run.store, run.stats


def plan_sha(plan) -> str:
    """Digest of one plan in the encoding of tests/golden/make_golden.py."""
    iteration, pf, uniq, ttl, _, lk = plan
    h = hashlib.sha256()
    h.update(np.asarray([iteration, lk, len(pf), len(uniq)], dtype="<i8").tobytes())
    h.update(np.asarray(pf, dtype="<u8").tobytes())
    h.update(np.asarray(uniq, dtype="<u8").tobytes())
    h.update(np.asarray(ttl, dtype="<i8").tobytes())
    return h.hexdigest()
