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


def _bits(a) -> list:
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).tolist()


def _b64(a, dtype) -> str:
    import base64

    return base64.b64encode(np.ascontiguousarray(a, dtype=dtype).tobytes()).decode()


def gen_api():
    """Pins of the remaining public API rows: DynamicCache
    content_checksum / canonical_digest / evict_expired / drain
    (cache.py:214-286), the trainer object wrappers (trainer.py:56-179),
    ShardedStore.shard_of (store.py:80-88) and the plan text format with the
    CLI's worked-example records (lookahead.py:162-189, tests/test_cli.py:97-103).
    Every input of a scenario is recorded next to its outputs, so the tests
    replay exactly these operations."""
    from embcache.cache import DynamicCache
    from embcache.lookahead import parse_plan
    from embcache.store import ShardedStore
    from embcache.trainer import (StubModelConfig, apply_updates, combine_gradients, local_gradients,
                                  split_sync_sets)

    out = {}
    rng = np.random.default_rng(2024)

    def cache_state(c, compact=False):
        st = {"len": len(c), "checksum": c.content_checksum(), "digest": c.canonical_digest()}
        if not compact:
            keys = sorted(c.key_set())
            st.update(ttl=[c.ttl_of(k) for k in keys], dirty=[c.is_dirty(k) for k in keys],
                      keys=[packed(k) for k in keys])
        return st

    def released(items, compact):
        if compact:  # large scenario: count + sha256 over (keys u64, value bits, dirty u8)
            return {"n": len(items), "sha": sha(np.asarray([packed(k) for k, _, _ in items], dtype="<u8"),
                                                 np.asarray([v for _, v, _ in items], dtype="<f4"),
                                                 np.asarray([d for _, _, d in items], dtype=np.uint8))}
        return [[packed(k), _bits(v), bool(d)] for k, v, d in items]

    # -- cache scenarios: a small hand-sized one and a 3,000-entry one
    for name, cap, dim, n, tables in (("small", 16, 4, 9, 3), ("large", 4096, 16, 2000, 5)):
        c = DynamicCache(cap, dim)
        keyset = set()
        while len(keyset) < n:
            keyset.add((int(rng.integers(0, tables)), int(rng.integers(0, 50 * n))))
        keys = sorted(EmbeddingKey(t, r) for t, r in keyset)
        vals = rng.standard_normal((n, dim)).astype(np.float32)
        ttls = rng.integers(0, 6, size=n).tolist()
        half = n // 2
        ops = {"keys": [packed(k) for k in keys], "values": _b64(vals, "<f4"), "ttls": ttls, "half": half}
        c.apply_prefetch(keys[:half], vals[:half], {k: t for k, t in zip(keys[:half], ttls[:half])})
        c.apply_prefetch(keys[half:], vals[half:], {k: t for k, t in zip(keys[half:], ttls[half:])})
        sc = {"capacity": cap, "dim": dim, "ops": ops, "after_prefetch": cache_state(c, name == "large")}
        upd_idx = sorted(rng.choice(n, size=max(1, n // 3), replace=False).tolist())
        new_ttl = rng.integers(2, 9, size=len(upd_idx)).tolist()
        c.apply_ttl_updates([(keys[i], t) for i, t in zip(upd_idx, new_ttl)])
        ops["ttl_updates"] = [upd_idx, new_ttl]
        row_idx = sorted(rng.choice(n, size=max(1, n // 2), replace=False).tolist())
        slots = c.resolve_slots([keys[i] for i in row_idx])
        new_rows = rng.standard_normal((len(row_idx), dim)).astype(np.float32)
        mask = rng.integers(0, 2, size=len(row_idx)).astype(bool)
        c.update_rows(slots, new_rows, mask)
        ops["update_rows"] = [row_idx, _b64(new_rows, "<f4"), mask.astype(int).tolist()]
        wl = keys[n - 1]
        wl_val = rng.standard_normal(dim).astype(np.float32)
        c.write_local_update(wl, wl_val)
        ops["write_local"] = [n - 1, _bits(wl_val)]
        sc["after_update"] = cache_state(c, name == "large")
        sc["evict_2"] = released(c.evict_expired(2), name == "large")
        sc["after_evict"] = cache_state(c, name == "large")
        sc["drain"] = released(c.drain(), name == "large")
        sc["after_drain"] = cache_state(c, name == "large")
        sc["counters"] = {"insertions": c.insertions, "evictions": c.evictions, "peak": c.peak_occupancy}
        out[f"cache_{name}"] = sc

    # -- trainer object wrappers (3 ranks, overlapping keys, one empty rank)
    cfgm = StubModelConfig(lr=0.05, c_value=0.01, c_label=0.001)
    dim = 4
    universe = [EmbeddingKey(t, r) for t in range(2) for r in range(6)]
    values = {k: rng.standard_normal(dim).astype(np.float32) for k in universe}
    ranks = []
    for r in range(3):
        exs = []
        for i in range(0 if r == 1 else 5):
            sparse = tuple(universe[j] for j in rng.choice(len(universe), size=2, replace=False))
            exs.append(Example(int(rng.integers(0, 2)), (), sparse))
        ranks.append(exs)
    per_trainer = [local_gradients(exs, values, cfgm) for exs in ranks]
    combined = combine_gradients(per_trainer)
    c = DynamicCache(32, dim)
    ukeys = sorted(values)
    c.apply_prefetch(ukeys, np.stack([values[k] for k in ukeys]), {k: 9 for k in ukeys})
    # one zero-gradient key: must stay clean (trainer.py:149-165)
    zero_key = next(k for k in ukeys if k not in combined)
    combined_z = dict(combined)
    combined_z[zero_key] = np.zeros(dim, dtype=np.float32)
    updated = apply_updates(c, combined_z, cfgm)
    nxt = set(universe[::3])
    crit, bg = split_sync_sets(updated, nxt)
    out["trainer"] = {
        "cfg": [cfgm.lr, cfgm.c_value, cfgm.c_label], "dim": dim,
        "values": [[packed(k), _bits(values[k])] for k in ukeys],
        "ranks": [[[ex.label, [packed(k) for k in ex.sparse]] for ex in exs] for exs in ranks],
        "local": [[[packed(k), _bits(v)] for k, v in g.items()] for g in per_trainer],
        "combined": [[packed(k), _bits(v)] for k, v in combined.items()],
        "zero_key": packed(zero_key), "updated": sorted(packed(k) for k in updated),
        "after_apply": cache_state(c),
        "next": sorted(packed(k) for k in nxt), "critical": [packed(k) for k in crit],
        "background": [packed(k) for k in bg]}

    # -- shard placement
    schema = Schema(4, (1000, 50, 7, 100000), 0, 4)
    tk = [(int(rng.integers(0, 4)), 0) for _ in range(40)]
    tk = [(t, int(rng.integers(0, schema.rows_per_table[t]))) for t, _ in tk]
    out["shard_of"] = {"schema": [4, list(schema.rows_per_table), 0, 4], "keys": [packed(EmbeddingKey(*x)) for x in tk],
                       "shards": {str(ns): [ShardedStore(schema, ns, 3).shard_of(EmbeddingKey(*x)) for x in tk]
                                  for ns in (1, 3, 4, 7, 16)}}

    # -- plan text format: the CLI worked-example records and the small fixture
    worked = [make_batch(1, [3, 9]), make_batch(2, [3, 4]), make_batch(3, [3, 6]), make_batch(4, [1, 6])]
    wplans, _ = plan_stream(worked, 2, 100)
    _, small = small_fixture()
    splans, _ = plan_stream(small, 8, 5000)
    lines = [format_plan(p) for p in splans[:12]]
    parsed = [plan_record(parse_plan(ln)) for ln in lines]
    out["plan_text"] = {"worked": [format_plan(p) for p in wplans], "small_L8": lines, "small_L8_parsed": parsed,
                        "empty": format_plan(parse_plan("iter=7 prefetch= ttl="))}
    dump("api.json", out)


def gen_cli():
    """Outputs of the reference CLI itself (reference cli.py; fixtures of
    tests/test_cli.py:22-51): gen-trace file bytes, plan records, run /
    baseline report bytes and stdout, verify exit codes."""
    import contextlib
    import io
    import tempfile

    from embcache.cli import main as cli_main
    from embcache.traces import write_trace

    def call(argv):
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = cli_main(argv)
        return rc, buf.getvalue()

    out = {}
    with tempfile.TemporaryDirectory() as td:
        gen = os.path.join(td, "gen.trace")
        rc, so = call(["gen-trace", "--schema", "2:300,200:1:4", "--zipf", "1.05", "--examples", "500", "--seed", "3",
                       "--out", gen])
        out["gen_trace"] = {"rc": rc, "stdout": so, "sha256": hashlib.sha256(open(gen, "rb").read()).hexdigest()}
        zipf = os.path.join(td, "zipf.trace")
        schema = Schema(2, (600, 400), 2, 4)
        write_trace(zipf, schema, generate_synthetic_trace(ZipfSpec(schema, 1.05, 30 * 64, seed=7)))
        worked = os.path.join(td, "fig.trace")
        wb = [make_batch(1, [3, 9]), make_batch(2, [3, 4]), make_batch(3, [3, 6]), make_batch(4, [1, 6])]
        write_trace(worked, Schema(1, (10,), 0, 4), [ex for b in wb for ex in b.examples])
        plans = os.path.join(td, "plans.txt")
        rc, so = call(["plan", "--trace", worked, "--batch-size", "2", "--lookahead", "2", "--capacity", "100",
                       "--first-iteration", "1", "--out", plans])
        out["plan_worked"] = {"rc": rc, "stdout": so, "lines": open(plans).read().splitlines()}
        rc, so = call(["plan", "--trace", zipf, "--batch-size", "64", "--lookahead", "8", "--capacity", "5000",
                       "--out", plans])
        out["plan_zipf"] = {"rc": rc, "stdout": so, "sha256": hashlib.sha256(open(plans, "rb").read()).hexdigest(),
                            "first": open(plans).read().splitlines()[:3]}
        cfg = os.path.join(td, "config.json")
        with open(cfg, "w") as fh:
            json.dump(dict(cache_capacity=5_000, batch_size=64, lookahead=8, num_trainers=2, seed=5), fh)
        reports = {}
        for cmd in ("run", "baseline"):
            rep = os.path.join(td, f"{cmd}.json")
            rc, so = call([cmd, "--config", cfg, "--trace", zipf, "--report", rep, "--dump-store"])
            reports[cmd] = rep
            out[cmd] = {"rc": rc, "stdout": so, "json": open(rep).read(),
                        "csv": open(rep[:-5] + ".csv").read(),
                        "store_sha256": hashlib.sha256(open(rep[:-5] + ".store", "rb").read()).hexdigest()}
        rc, so = call(["verify", "--a", reports["run"], "--b", reports["baseline"]])
        out["verify"] = {"rc": rc, "stdout": so}
    dump("cli.json", out)


def gen_wire():
    """Frames of the reference store protocol (reference wire.py) and a served
    session transcript against a fresh store (schema 2:(1000,300):0:4, 3
    shards, seed 11): request bytes in, response bytes out."""
    import io

    from embcache import wire as W

    keys = [EmbeddingKey(0, 3), EmbeddingKey(1, 299), EmbeddingKey(0, 999), EmbeddingKey(1, 0)]
    vals = (np.arange(16, dtype=np.float32).reshape(4, 4) * 0.25 - 1.0)
    out = {"fetch": W.encode_fetch(keys).hex(), "fetch_resp": W.encode_fetch_resp(vals).hex(),
           "write": W.encode_write(keys, vals).hex(), "ack": W.encode_ack(7).hex(),
           "keys": [[k.table_id, k.row_id] for k in keys], "values": _bits(vals)}
    schema = Schema(2, (1000, 300), 0, 4)
    store = ShardedStore(schema, 3, 11)
    reqs = (W.encode_fetch(keys) + W.encode_write(keys[:2], vals[:2]) + W.encode_fetch(keys)
            + W.encode_fetch([EmbeddingKey(1, 5)]))
    wbuf = io.BytesIO()
    served = W.serve_connection(store, io.BytesIO(reqs), wbuf)
    out["session"] = {"schema": [2, [1000, 300], 0, 4], "num_shards": 3, "seed": 11, "requests": reqs.hex(),
                      "responses": wbuf.getvalue().hex(), "served": served}
    dump("wire.json", out)


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
    if want("api"):
        gen_api()
    if want("cli"):
        gen_cli()
    if want("wire"):
        gen_wire()
    if want("acceptance"):
        gen_acceptance()
    ck = gen_ck() if want("ck") else None
    if want("generator"):
        gen_generator(ck)


if __name__ == "__main__":
    sys.exit(main())
