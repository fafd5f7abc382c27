"""Generate the golden fixtures under tests/golden/ from the REFERENCE package.

Run only in the build container, where the reference is importable:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py [--skip-ck]

Everything written here is an output of the reference itself (reference
``pkg/src/embcache``): generator stream digests, plan streams, engine reports
(JSON + CSV bytes), final store digests, fault outcomes.  The GPU box never
reads /root/reference; tests only read these committed files.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

import embcache  # noqa: F401  (the reference; PYTHONPATH must point at it)
from embcache.engine import EngineConfig, run_pipeline, run_synchronous_baseline
from embcache.errors import CacheMissError
from embcache.lookahead import format_plan, new_state, emit_next_plan, adapt_on_pressure
from embcache.store import ShardedStore, initial_values
from embcache.hashing import fnv1a64_u64s, splitmix64
from embcache.traces import Batch, EmbeddingKey, Example, Schema, ZipfSpec, batchify, generate_synthetic_trace

HERE = os.path.dirname(os.path.abspath(__file__))

CK_ROWS = (1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683, 8351593, 3194, 27,
           14992, 5461306, 10, 5652, 2173, 4, 7046547, 18, 15, 286181, 105, 142572)


def packed(key) -> int:
    return (int(key[0]) << 44) | int(key[1])


def columns_of(batches):
    rows = np.asarray([[k.row_id for k in ex.sparse] for b in batches for ex in b.examples], dtype=np.int64)
    labels = np.asarray([ex.label for b in batches for ex in b.examples], dtype=np.uint8)
    dense = np.asarray([ex.dense for b in batches for ex in b.examples], dtype=np.float32)
    return rows, labels, dense


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def plan_record(plan) -> list:
    return [plan.iteration, plan.lookahead, [packed(k) for k in plan.prefetch],
            [[packed(k), t] for k, t in plan.ttl_updates]]


def plan_sha(plan) -> str:
    pf = np.asarray([packed(k) for k in plan.prefetch], dtype="<u8")
    tk = np.asarray([packed(k) for k, _ in plan.ttl_updates], dtype="<u8")
    tv = np.asarray([t for _, t in plan.ttl_updates], dtype="<i8")
    head = np.asarray([plan.iteration, plan.lookahead, len(pf), len(tk)], dtype="<i8")
    return sha(head, pf, tk, tv)


def plan_stream(batches, lookahead, capacity):
    state = new_state(lookahead, capacity)
    src = iter(batches)
    plans = []
    while (p := emit_next_plan(state, src)) is not None:
        plans.append(p)
        adapt_on_pressure(state)
    stats = dict(lookahead=state.lookahead, insertions=state.insertions, removals=state.removals,
                 peak_occupancy=state.peak_occupancy, peak_projected=state.peak_projected)
    return plans, stats


def report_blob(report) -> dict:
    return {"json": report.to_json_bytes().decode(), "csv": report.to_csv_bytes().decode()}


def dump(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w") as fh:
        json.dump(obj, fh, sort_keys=True, separators=(",", ":"))
        fh.write("\n")
    print(f"wrote {path} ({os.path.getsize(path)} bytes)", flush=True)


def small_fixture():
    schema = Schema(2, (600, 400), 2, 4)
    spec = ZipfSpec(schema, 1.05, 60 * 64, seed=7)
    return schema, list(batchify(generate_synthetic_trace(spec), 64))


def make_batch(iteration, rows, table=0):
    return Batch(iteration, [Example(i & 1, (), (EmbeddingKey(table, r),)) for i, r in enumerate(rows)])


def gen_hashing():
    out = {"fnv_bytes": [[s, hex(__import__("embcache.hashing", fromlist=["fnv1a64"]).fnv1a64(s.encode()))]
                         for s in ("", "a", "foobar")]}
    rng = np.random.default_rng(5)
    words = rng.integers(0, 2**63, size=(16, 3), dtype=np.int64).tolist()
    out["fnv_u64s"] = [[w, fnv1a64_u64s(*w)] for w in words]
    out["splitmix"] = [[x, splitmix64(x)] for x in (0, 1, 1234567, 2**64 - 1, 0x9E3779B97F4A7C15)]
    schema = Schema(3, (7, 50000, 3), 0, 16)
    tables = np.asarray([0, 1, 1, 2, 0, 1], dtype=np.int64)
    rows = np.asarray([0, 12345, 49999, 2, 6, 0], dtype=np.int64)
    out["init"] = []
    for seed in (0, 11, 99, 2**63 + 5):
        vals = initial_values(schema, seed, tables, rows)
        out["init"].append([seed, tables.tolist(), rows.tolist(), vals.view(np.uint32).tolist()])
    dump("hashing.json", out)


def gen_generator(ck_batches=None):
    out = {}
    for name, schema, s, n, seed in (
        ("small", Schema(2, (600, 400), 2, 4), 1.05, 3840, 7),
        ("mixed", Schema(3, (7, 5000, 3), 1, 4), 0.8, 5000, 42),
        ("acceptance", Schema(2, (60000, 40000), 2, 4), 1.05, 256000, 1337),
    ):
        exs = list(generate_synthetic_trace(ZipfSpec(schema, s, n, seed)))
        rows = np.asarray([[k.row_id for k in ex.sparse] for ex in exs], dtype=np.int64).reshape(n, schema.num_tables)
        labels = np.asarray([ex.label for ex in exs], dtype=np.uint8)
        dense = np.asarray([ex.dense for ex in exs], dtype=np.float32).reshape(n, schema.num_dense)
        out[name] = {"schema": [schema.num_tables, list(schema.rows_per_table), schema.num_dense, schema.emb_dim],
                     "exponent": s, "n": n, "seed": seed,
                     "rows_sha": sha(rows), "labels_sha": sha(labels), "dense_sha": sha(dense)}
    if ck_batches is not None:
        rows, labels, dense = columns_of(ck_batches)
        out["ck12"] = {"schema": [26, list(CK_ROWS), 13, 16], "exponent": 1.05, "n": len(labels), "seed": 1,
                       "rows_sha": sha(rows), "labels_sha": sha(labels), "dense_sha": sha(dense)}
    dump("generator.json", out)


def cfg_small(**kw):
    base = dict(cache_capacity=5000, batch_size=64, lookahead=8, num_trainers=1, num_shards=2, seed=5,
                replication_check_interval=1, check_mirror=True)
    base.update(kw)
    return EngineConfig(**base)


def gen_planner_and_engine():
    schema, batches = small_fixture()
    plans = {}
    for lookahead, cap in ((8, 10**6), (1, 10**6), (16, 5000), (32, 550), (3, 10**6)):
        ps, stats = plan_stream(batches, lookahead, cap)
        plans[f"L{lookahead}_cap{cap}"] = {"lookahead": lookahead, "capacity": cap,
                                           "plans": [plan_record(p) for p in ps], "stats": stats}
    worked = [make_batch(1, [3, 9]), make_batch(2, [3, 4]), make_batch(3, [3, 6]), make_batch(4, [1, 6])]
    ps, stats = plan_stream(worked, 2, 100)
    plans["worked_L2"] = {"lookahead": 2, "capacity": 100, "plans": [plan_record(p) for p in ps], "stats": stats}
    dump("plans_small.json", plans)

    reports = {}
    cases = {
        "L8_T1": dict(),
        "L4_T3_rpc1": dict(lookahead=4, num_trainers=3, rpc_batch_proportion=1.0),
        "L32_cap550_halving": dict(lookahead=32, cache_capacity=550),
        "auto_cap900": dict(lookahead=0, cache_capacity=900),
        "L8_nosplit": dict(split_sync=False),
        "L16_T2": dict(lookahead=16, num_trainers=2),
        "L1_T2_rpc1": dict(lookahead=1, num_trainers=2, rpc_batch_proportion=1.0),
        "L8_T1_events": dict(record_events=True),
    }
    for name, kw in cases.items():
        rep = run_pipeline(cfg_small(**kw), schema, batches)
        blob = report_blob(rep)
        if rep.events is not None:
            blob["events"] = [{"iteration": e["iteration"], "prefetch": [packed(k) for k in e["prefetch"]],
                               "ttl_updates": [[packed(k), t] for k, t in e["ttl_updates"]],
                               "evicted": [packed(k) for k in e["evicted"]]} for e in rep.events]
        blob["config"] = cfg_small(**kw).to_dict()
        reports[name] = blob
    for trainers in (1, 2, 3):
        rep = run_synchronous_baseline(cfg_small(num_trainers=trainers), schema, batches)
        reports[f"baseline_T{trainers}"] = dict(report_blob(rep), config=cfg_small(num_trainers=trainers).to_dict())
    # Faults: the miss carries key + iteration; the ungated run's stale digest.
    try:
        run_pipeline(cfg_small(), schema, batches, fault="drop_prefetch")
        raise SystemExit("drop_prefetch did not raise")
    except CacheMissError as err:
        reports["fault_drop_prefetch"] = {"key": packed(err.key), "iteration": err.iteration}
    stale = run_pipeline(cfg_small(check_mirror=False), schema, batches, fault="no_gate")
    reports["fault_no_gate"] = dict(report_blob(stale), config=cfg_small(check_mirror=False).to_dict())
    # Worked example (tests/test_engine.py:53-71 shape) with events.
    wschema = Schema(1, (10,), 0, 4)
    wcfg = cfg_small(lookahead=2, batch_size=2, cache_capacity=100, record_events=True)
    rep = run_pipeline(wcfg, wschema, worked)
    blob = report_blob(rep)
    blob["evicted"] = [[packed(k) for k in e["evicted"]] for e in rep.events]
    blob["config"] = wcfg.to_dict()
    reports["worked"] = blob
    dump("reports_small.json", reports)


def gen_acceptance():
    schema = Schema(2, (60_000, 40_000), 2, 4)
    spec = ZipfSpec(schema, 1.05, 500 * 512, seed=1337)
    t0 = time.time()
    batches = list(batchify(generate_synthetic_trace(spec), 512))
    print(f"acceptance trace {time.time() - t0:.1f}s", flush=True)

    def cfg(trainers, lookahead, rpc, cap, **kw):
        d = dict(cache_capacity=cap, batch_size=512, lookahead=lookahead, num_trainers=trainers,
                 num_shards=4, rpc_batch_proportion=rpc, seed=11)
        d.update(kw)
        return EngineConfig(**d)

    out = {"baseline": {}, "pipeline": {}}
    for t in (1, 2, 4):
        rep = run_synchronous_baseline(cfg(t, 1, 0.25, 50_000), schema, batches,
                                       trace_fingerprint="zipf1337/512x500")
        out["baseline"][str(t)] = rep.final_store_digest
        print("baseline", t, rep.final_store_digest, flush=True)
    for t, lk, rpc, cap in ((2, 64, 0.25, 16_000), (4, 200, 1.0, 16_000), (1, 8, 0.25, 50_000)):
        c = cfg(t, lk, rpc, cap)
        rep = run_pipeline(c, schema, batches, trace_fingerprint="zipf1337/512x500")
        out["pipeline"][f"T{t}_L{lk}_rpc{rpc}_cap{cap}"] = dict(report_blob(rep), config=c.to_dict())
        print("pipeline", t, lk, rep.final_store_digest, flush=True)
    dump("acceptance.json", out)


def gen_ck(iterations=12):
    schema = Schema(26, CK_ROWS, 13, 16)
    t0 = time.time()
    spec = ZipfSpec(schema, 1.05, iterations * 16384, seed=1)
    batches = list(batchify(generate_synthetic_trace(spec), 16384))
    print(f"ck trace {time.time() - t0:.1f}s", flush=True)
    cap = schema.total_rows // 100
    out = {"capacity": cap, "iterations": iterations}
    plans, stats = plan_stream(batches, 7, cap)
    out["plans_L7"] = {"sha": [plan_sha(p) for p in plans], "prefetch": [len(p.prefetch) for p in plans],
                       "unique": [len(p.ttl_updates) for p in plans], "stats": stats,
                       "first_plan_head": plan_record(plans[0])[:2] + [plan_record(plans[0])[2][:64]]}
    c = EngineConfig(cache_capacity=cap, batch_size=16384, lookahead=0, num_trainers=1, num_shards=1, seed=11)
    t0 = time.time()
    rep = run_pipeline(c, schema, batches)
    print(f"ck pipeline {time.time() - t0:.1f}s {rep.final_store_digest}", flush=True)
    out["pipeline_T1"] = dict(report_blob(rep), config=c.to_dict())
    c8 = EngineConfig(cache_capacity=cap, batch_size=16384, lookahead=0, num_trainers=8, num_shards=1, seed=11)
    t0 = time.time()
    rep8 = run_synchronous_baseline(c8, schema, batches)
    print(f"ck baseline T8 {time.time() - t0:.1f}s {rep8.final_store_digest}", flush=True)
    out["baseline_T8_digest"] = rep8.final_store_digest
    dump("ck12.json", out)
    return batches


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    only = set(filter(None, args.only.split(",")))
    want = lambda name: not only or name in only  # noqa: E731
    if want("hashing"):
        gen_hashing()
    if want("engine"):
        gen_planner_and_engine()
    if want("acceptance"):
        gen_acceptance()
    ck = gen_ck() if want("ck") else None
    if want("generator"):
        gen_generator(ck)


if __name__ == "__main__":
    sys.exit(main())
