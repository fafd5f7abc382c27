"""The CPU oracle is pinned to golden vectors produced by the reference itself.

Golden sources: tests/golden/*.json (tests/golden/make_golden.py ran the
reference package).  Nothing here needs a GPU.
"""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import golden, make_batch, unpack
from oracle import bagpipe_oracle as O
from paper_2202_12429_b200.traces import Schema, ZipfSpec, batchify_columns, generate_columns


def test_hash_vectors():
    g = golden("hashing.json")
    for words, want in g["fnv_u64s"]:
        assert int(O.fnv_cols(*[np.asarray([w], dtype=np.uint64) for w in words])[0]) == want
    for x, want in g["splitmix"]:
        assert int(O.splitmix(np.asarray([x], dtype=np.uint64))[0]) == want


def test_init_values_match_reference():
    g = golden("hashing.json")
    for seed, tables, rows, bits in g["init"]:
        got = O.init_rows(seed, tables, rows, 16)
        assert got.view(np.uint32).tolist() == bits


def _plans_equal(got, want):
    assert len(got) == len(want)
    for (it, pf, uniq, ttl, _, lk), (wit, wlk, wpf, wttl) in zip(got, want):
        assert it == wit and lk == wlk
        assert pf.tolist() == wpf
        assert [[int(k), int(t)] for k, t in zip(uniq, ttl)] == wttl


def test_worked_example_plans():
    g = golden("plans_small.json")["worked_L2"]
    batches = [make_batch(1, [3, 9]), make_batch(2, [3, 4]), make_batch(3, [3, 6]), make_batch(4, [1, 6])]
    plans, stats = O.plan_stream(batches, 2, 100)
    _plans_equal(plans, g["plans"])
    assert stats == g["stats"]


@pytest.mark.parametrize("case", ["L8_cap1000000", "L1_cap1000000", "L16_cap5000", "L32_cap550", "L3_cap1000000"])
def test_small_fixture_plan_streams(small_batches, case):
    g = golden("plans_small.json")[case]
    plans, stats = O.plan_stream(small_batches, g["lookahead"], g["capacity"])
    _plans_equal(plans, g["plans"])
    assert stats == g["stats"]


def _cfg(report):
    return json.loads(report["json"])


def test_small_fixture_baseline_digests(small_schema, small_batches):
    reports = golden("reports_small.json")
    for t in (1, 2, 3):
        want = _cfg(reports[f"baseline_T{t}"])["final_store_digest"]
        store = O.baseline(small_batches, small_schema.rows_per_table, 4, 5, t)
        assert store.digest() == want


@pytest.mark.parametrize("case", ["L8_T1", "L4_T3_rpc1", "L32_cap550_halving", "L16_T2", "L1_T2_rpc1"])
def test_small_fixture_pipeline_digests(small_schema, small_batches, case):
    rep = golden("reports_small.json")[case]
    c = rep["config"]
    store, stats = O.pipeline(small_batches, small_schema.rows_per_table, 4, c["seed"], c["num_trainers"],
                              c["cache_capacity"], c["lookahead"], c["rpc_batch_proportion"])
    summary = _cfg(rep)
    assert store.digest() == summary["final_store_digest"]
    rows = rep["csv"].strip().split("\n")[1:]
    for st, row in zip(stats, rows):
        cells = row.split(",")
        assert st["occupancy_peak"] == int(cells[7]) and st["occupancy_end"] == int(cells[8])
        assert st["prefetch"] == int(cells[10]) and st["evicted"] == int(cells[11])


def test_acceptance_baseline_t1_digest():
    """The frozen oracle fixture of reference tests/test_acceptance.py:64."""
    schema = Schema(2, (60_000, 40_000), 2, 4)
    rows, labels, dense = generate_columns(ZipfSpec(schema, 1.05, 500 * 512, seed=1337))
    batches = batchify_columns(rows, labels, dense, 512)
    store = O.baseline(batches, schema.rows_per_table, 4, 11, 1)
    assert store.digest() == "f2c6d9f7b649188cce3461885f54dacd"
    assert golden("acceptance.json")["baseline"]["1"] == "f2c6d9f7b649188cce3461885f54dacd"


def test_ck_plan_stream_digests():
    """Criteo-Kaggle shape, 12 batches of 16,384 at L=7, capacity 1% of rows:
    per-plan digests recorded from the reference planner."""
    g = golden("ck12.json")
    gen = golden("generator.json")["ck12"]
    nt, rpt, nd, dim = gen["schema"]
    rows, labels, dense = generate_columns(ZipfSpec(Schema(nt, rpt, nd, dim), gen["exponent"], gen["n"], gen["seed"]))
    batches = batchify_columns(rows, labels, None, 16384)
    plans, stats = O.plan_stream(batches, 7, g["capacity"])
    assert stats == g["plans_L7"]["stats"]
    for p, sha, npf in zip(plans, g["plans_L7"]["sha"], g["plans_L7"]["prefetch"]):
        assert len(p[1]) == npf
        assert O.plan_sha(p) == sha
