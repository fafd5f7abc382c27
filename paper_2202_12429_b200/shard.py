"""Table-wise and row-wise sharding of the embedding path across GPUs (one
process per GPU).

Every key belongs to exactly one table, and every per-key decision of the
path -- Algorithm 1's TTLs and prefetches, the cache, the stub gradient's
per-key sequential sums -- depends only on that key's occurrences.  Giving
each rank a disjoint set of tables (the full global batch restricted to them,
keys keeping their global table ids, so the functional initial values are
unchanged) partitions the work without any data-path collective, and the
union of the shard stores equals the single-GPU store bit for bit
(tests/test_shard_dist.py checks it with gloo on CPU ranks).

Tables are dealt round-robin by default: every table contributes exactly one
key per example, so ranks differ by at most one table's worth of
occurrences.  With a per-table cost (e.g. unique keys per batch, which drive
prefetch, insertion, eviction and the trainer) the tables are instead dealt
longest-processing-time first, each to the rank with the least cost so far.

Row-wise sharding (row_shard_batches) places every KEY by the reference
store's own placement hash, fnv1a64(table, row) mod N (reference
store.py:80-88, 100-104): a 10M-row table is spread over all ranks instead of
landing on one.  A rank's batch holds, example by example, the occurrences of
its keys (an occurrence-backed Batch: examples carry a variable number of
keys), so each key keeps all of its occurrences in occurrence order and every
trainer rank (example index / (B/T), engine.py:159-161) keeps its examples --
the same per-key arithmetic as one GPU, exact by the same argument.
"""

from __future__ import annotations

import numpy as np

from .traces import Batch


def table_shards(num_tables: int, world: int, cost=None) -> list:
    """Tables owned by each rank, in increasing table order: round-robin, or
    greedy by ``cost[t]`` (largest first, to the least-loaded rank; ties to
    the lower rank) -- deterministic, so every rank computes the same split."""
    if cost is None:
        return [list(range(r, num_tables, world)) for r in range(world)]
    cost = np.asarray(cost, dtype=np.float64)
    if cost.shape != (num_tables,):
        raise ValueError("cost needs one entry per table")
    load = np.zeros(world)
    out = [[] for _ in range(world)]
    for t in sorted(range(num_tables), key=lambda t: (-cost[t], t)):
        r = int(np.argmin(load))
        out[r].append(t)
        load[r] += cost[t]
    return [sorted(ts) for ts in out]


def table_costs(batch: Batch, unique_weight: float = 4.0) -> np.ndarray:
    """Sharding cost per table of one columnar batch: its occurrences (one per
    example: batch prep, trainer streams) plus ``unique_weight`` x its unique
    keys (lookups, prefetches, insertions, evictions, write-back)."""
    if not batch.is_columnar:
        raise ValueError("table costs need a columnar batch")
    n = batch.rows.shape[0]
    return np.asarray([n + unique_weight * len(np.unique(batch.rows[:, c])) for c in range(batch.rows.shape[1])],
                      dtype=np.float64)


def shard_batches(batches: list, tables: list) -> list:
    """Column-restricted columnar batches holding the rank's tables of every example."""
    out = []
    for b in batches:
        if not b.is_columnar:
            raise ValueError("sharding needs columnar batches (batchify_columns / read_trace_columns)")
        cols = [int(np.flatnonzero(b.table_ids() == t)[0]) for t in tables]
        out.append(Batch.from_columns(b.iteration, np.ascontiguousarray(b.rows[:, cols]), b.labels, b.dense,
                                      tables=tables))
    return out


def row_owner(keys: np.ndarray, world: int) -> np.ndarray:
    """Owning rank of every packed key: fnv1a64(table, row) mod world, the
    reference store's shard placement (store.py:80-88)."""
    from .store import shard_of_keys

    keys = np.asarray(keys, dtype=np.uint64)
    return shard_of_keys(keys >> np.uint64(44), keys & np.uint64((1 << 44) - 1), world)


def row_shard_batches(batches: list, world: int, rank: int) -> list:
    """The rank's occurrences of every batch (keys with row_owner == rank), in
    occurrence order, as occurrence-backed batches with the original example
    boundaries (so trainer ranks are unchanged)."""
    out = []
    for b in batches:
        keys, labels, offsets = b.packed_occurrences()
        mine = row_owner(keys, world) == rank
        per_ex = np.add.reduceat(mine.astype(np.int64), offsets[:-1]) if keys.size else np.zeros(0, np.int64)
        # reduceat repeats the value at empty examples: zero them
        per_ex = np.where(offsets[1:] > offsets[:-1], per_ex, 0)
        offs = np.zeros(offsets.size, dtype=np.int64)
        np.cumsum(per_ex, out=offs[1:])
        out.append(Batch.from_occurrences(b.iteration, keys[mine], labels[mine], offs))
    return out


def owned_rows(schema, tables: list) -> np.ndarray:
    """Global row indices g of the rank's tables (to reassemble full stores)."""
    base = schema.table_base()
    return np.concatenate([np.arange(base[t], base[t + 1]) for t in tables]) if tables else np.zeros(0, np.int64)
