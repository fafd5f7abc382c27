"""GPU engine vs the reference: byte-identical reports, bit-exact digests,
fault detection (reference tests/test_engine.py, tests/test_acceptance.py
criteria 2, 3, 6).  Golden reports were produced by the reference."""

from __future__ import annotations

import json

import pytest

from conftest import golden, unpack
from oracle import bagpipe_oracle as O
from paper_2202_12429_b200.traces import Batch, Schema, ZipfSpec, batchify_columns, generate_columns

pytestmark = pytest.mark.gpu

SMALL_CASES = ["L8_T1", "L4_T3_rpc1", "L32_cap550_halving", "auto_cap900", "L8_nosplit", "L16_T2", "L1_T2_rpc1",
               "L8_T1_events"]


def _engine():
    from paper_2202_12429_b200 import engine

    return engine


def _cfg(d):
    return _engine().EngineConfig.from_dict(d)


def _assert_report(report, blob):
    assert report.to_json_bytes().decode() == blob["json"]
    assert report.to_csv_bytes().decode() == blob["csv"]


@pytest.mark.parametrize("link_mode", [1, 2, 0])
@pytest.mark.parametrize("case", SMALL_CASES)
def test_pipeline_report_byte_identical(small_schema, small_batches, case, link_mode, monkeypatch):
    """Both host-link modes: copy engines + host pool (1), zero-copy kernels (0)."""
    monkeypatch.setenv("BAGPIPE_B200_LINK_MODE", str(link_mode))
    blob = golden("reports_small.json")[case]
    report = _engine().run_pipeline(_cfg(blob["config"]), small_schema, small_batches)
    _assert_report(report, blob)
    if "events" in blob:
        got = [{"iteration": e["iteration"], "prefetch": [(k[0] << 44) | k[1] for k in e["prefetch"]],
                "ttl_updates": [[(k[0] << 44) | k[1], t] for k, t in e["ttl_updates"]],
                "evicted": [(k[0] << 44) | k[1] for k in e["evicted"]]} for e in report.events]
        assert got == blob["events"]


@pytest.mark.parametrize("log_rows", ["0", "40", "700"])
@pytest.mark.parametrize("case", ["L8_T1", "L4_T3_rpc1", "L32_cap550_halving"])
def test_write_back_log_sizes(small_schema, small_batches, case, log_rows, monkeypatch):
    """Write-back log (DMA appends + commit, compaction when full): disabled
    (0: zero-copy scatter), smaller than most flush chunks (those fall back to
    the scatter, mixing both paths), and compacting every few flushes -- the
    report and digest stay byte-identical to the reference."""
    monkeypatch.setenv("BAGPIPE_B200_LOG_ROWS", log_rows)
    blob = golden("reports_small.json")[case]
    report = _engine().run_pipeline(_cfg(blob["config"]), small_schema, small_batches)
    _assert_report(report, blob)


@pytest.mark.parametrize("trainers", [1, 2, 3])
def test_baseline_report_byte_identical(small_schema, small_batches, trainers):
    blob = golden("reports_small.json")[f"baseline_T{trainers}"]
    report = _engine().run_synchronous_baseline(_cfg(blob["config"]), small_schema, small_batches)
    _assert_report(report, blob)


def test_object_batches_same_digest(small_schema, small_object_batches):
    blob = golden("reports_small.json")["L8_T1"]
    report = _engine().run_pipeline(_cfg(blob["config"]), small_schema, small_object_batches)
    assert report.final_store_digest == json.loads(blob["json"])["final_store_digest"]


def test_worked_example_event_log(worked_trace):
    blob = golden("reports_small.json")["worked"]
    report = _engine().run_pipeline(_cfg(blob["config"]), Schema(1, (10,), 0, 4), worked_trace)
    _assert_report(report, blob)
    assert [[(k[0] << 44) | k[1] for k in e["evicted"]] for e in report.events] == blob["evicted"]
    assert [[k.row_id for k in e["evicted"]] for e in report.events] == [[9], [4], [3], [1, 6]]


def test_dropped_prefetch_is_a_miss_at_the_reference_key(small_schema, small_batches):
    from paper_2202_12429_b200.errors import CacheMissError

    want = golden("reports_small.json")["fault_drop_prefetch"]
    cfg = _cfg(golden("reports_small.json")["L8_T1"]["config"])
    with pytest.raises(CacheMissError) as err:
        _engine().run_pipeline(cfg, small_schema, small_batches, fault="drop_prefetch")
    assert err.value.iteration == want["iteration"]
    assert err.value.key == unpack(want["key"])


@pytest.mark.parametrize("link_mode", [1, 2, 0])
def test_ungated_run_reproduces_reference_staleness(small_schema, small_batches, link_mode, monkeypatch):
    """fault=no_gate: the stale digest equals the reference's stale digest bit
    for bit, and differs from the baseline with a non-empty diff."""
    monkeypatch.setenv("BAGPIPE_B200_LINK_MODE", str(link_mode))
    eng = _engine()
    blob = golden("reports_small.json")["fault_no_gate"]
    cfg = _cfg(blob["config"])
    stale = eng.run_pipeline(cfg, small_schema, small_batches, fault="no_gate")
    _assert_report(stale, blob)
    base = eng.run_synchronous_baseline(cfg, small_schema, small_batches)
    result = eng.verify_equivalence(stale, base)
    assert not result.equal and result.diffs


@pytest.fixture(scope="module")
def acceptance_batches():
    schema = Schema(2, (60_000, 40_000), 2, 4)
    rows, labels, dense = generate_columns(ZipfSpec(schema, 1.05, 500 * 512, seed=1337))
    return schema, batchify_columns(rows, labels, dense, 512)


@pytest.mark.parametrize("trainers", [1, 2, 4])
def test_acceptance_baseline_digests(acceptance_batches, trainers):
    schema, batches = acceptance_batches
    eng = _engine()
    cfg = eng.EngineConfig(cache_capacity=50_000, batch_size=512, lookahead=1, num_trainers=trainers, num_shards=4,
                           seed=11)
    rep = eng.run_synchronous_baseline(cfg, schema, batches, trace_fingerprint="zipf1337/512x500")
    assert rep.final_store_digest == golden("acceptance.json")["baseline"][str(trainers)]


@pytest.mark.parametrize("case", ["T2_L64_rpc0.25_cap16000", "T4_L200_rpc1.0_cap16000", "T1_L8_rpc0.25_cap50000"])
def test_acceptance_pipeline_reports(acceptance_batches, case):
    schema, batches = acceptance_batches
    blob = golden("acceptance.json")["pipeline"][case]
    rep = _engine().run_pipeline(_cfg(blob["config"]), schema, batches, trace_fingerprint="zipf1337/512x500")
    _assert_report(rep, blob)


def test_ck12_pipeline_report_and_baseline_t8():
    """Criteo-Kaggle shape (config 2: cache 1% of rows, auto lookahead -> 7),
    12 iterations: report and final digest byte-identical to the reference;
    the T=8 synchronous baseline digest too."""
    eng = _engine()
    g = golden("ck12.json")
    gen = golden("generator.json")["ck12"]
    nt, rpt, nd, dim = gen["schema"]
    schema = Schema(nt, rpt, nd, dim)
    rows, labels, dense = generate_columns(ZipfSpec(schema, gen["exponent"], gen["n"], gen["seed"]))
    batches = batchify_columns(rows, labels, dense, 16384)
    rep = eng.run_pipeline(_cfg(g["pipeline_T1"]["config"]), schema, batches)
    _assert_report(rep, g["pipeline_T1"])
    cfg8 = eng.EngineConfig(cache_capacity=g["capacity"], batch_size=16384, lookahead=0, num_trainers=8,
                            num_shards=1, seed=11)
    assert eng.run_synchronous_baseline(cfg8, schema, batches).final_store_digest == g["baseline_T8_digest"]


@pytest.mark.parametrize("case", ["L8_T1", "L16_T2", "L32_cap550_halving", "auto_cap900"])
def test_threaded_planner_device_inputs_byte_identical(small_schema, small_batches, case):
    """The planner-thread path (device-resident batches, preps and plan
    emission on a second host thread) reproduces the reference reports."""
    import torch

    eng = _engine()
    blob = golden("reports_small.json")[case]
    cfg = _cfg(blob["config"])
    batches = eng._materialize(small_batches, cfg.iterations)
    dev = {}
    for i, b in enumerate(batches):
        keys, labels, _ = b.packed_occurrences()
        dev[i] = (torch.from_numpy(keys).cuda(), torch.from_numpy(labels).cuda())
    pipe = eng._Pipeline(cfg, small_schema, batches, None, None, device_inputs=dev, threaded=True)
    assert pipe._threaded
    report = pipe.run()
    _assert_report(report, blob)


@pytest.mark.parametrize("split", [True, False])
@pytest.mark.parametrize("rpc", [0.25, 1.0])
@pytest.mark.parametrize("capacity", [16_000, 50_000])
@pytest.mark.parametrize("lookahead", [1, 8, 64, 200])
@pytest.mark.parametrize("trainers", [1, 2, 4])
def test_acceptance_criterion2_matrix(acceptance_batches, trainers, lookahead, capacity, rpc, split):
    """Reference acceptance criteria 2 and 6 (tests/test_acceptance.py:142-153,
    258-267): the 48-cell matrix T x L x rpc x capacity, with and without the
    critical/background split, 500 iterations each, every pipelined digest
    bit-exact with the synchronous baseline (whose T=1 digest is the frozen
    f2c6d9f7...)."""
    schema, batches = acceptance_batches
    eng = _engine()
    cfg = eng.EngineConfig(cache_capacity=capacity, batch_size=512, lookahead=lookahead, num_trainers=trainers,
                           num_shards=4, seed=11, rpc_batch_proportion=rpc, split_sync=split)
    rep = eng.run_pipeline(cfg, schema, batches, trace_fingerprint="zipf1337/512x500")
    assert rep.final_store_digest == golden("acceptance.json")["baseline"][str(trainers)]


def test_threaded_mode_equals_serial(small_schema, small_batches):
    """mode="threaded" (reference engine.py:214-223) produces the serial
    run's records and digest (the reference asserts byte identity,
    tests/test_engine.py:275-299)."""
    import dataclasses
    import json as _json

    eng = _engine()
    cfg = _cfg(golden("reports_small.json")["L16_T2"]["config"])
    serial = eng.run_pipeline(cfg, small_schema, small_batches)
    threaded = eng.run_pipeline(dataclasses.replace(cfg, mode="threaded"), small_schema, small_batches)
    a, b = _json.loads(serial.to_json_bytes()), _json.loads(threaded.to_json_bytes())
    a["config"].pop("mode"), b["config"].pop("mode")
    assert a == b
    assert threaded.final_store_digest == serial.final_store_digest


@pytest.mark.parametrize("case", ["L8_T1", "L16_T2", "L32_cap550_halving"])
def test_pinned_host_batches_byte_identical(small_schema, case):
    """Batches in pinned host memory reproduce the reference reports: columnar
    batches through the compact upload (row-id planes of 4/2/1-byte columns
    + one label per example, expanded to packed keys on the GPU:
    bp_engine_add_batch_packed),
    object-backed ones through the pinned packed-occurrence DMA."""
    eng = _engine()
    blob = golden("reports_small.json")[case]
    cfg = _cfg(blob["config"])
    rows, labels, dense = generate_columns(ZipfSpec(small_schema, 1.05, 60 * 64, seed=7))
    columnar = [b.pin_memory() for b in batchify_columns(rows, labels, dense, 64)]
    assert all("pinned_planes" in b._memo for b in columnar)
    _assert_report(eng.run_pipeline(cfg, small_schema, columnar), blob)
    objects = [Batch(b.iteration, list(b.examples)).pin_memory() for b in batchify_columns(rows, labels, dense, 64)]
    assert all("pinned" in b._memo for b in objects)
    _assert_report(eng.run_pipeline(cfg, small_schema, objects), blob)


def test_pinned_planes_all_widths_equal_plain_run():
    """The compact upload with u8, u16 and u32 columns (tables of 200, 3,000
    and 100,000 rows): the same report bytes and store digest as the same
    batches uploaded as packed keys."""
    eng = _engine()
    schema = Schema(3, (200, 3000, 100000), 2, 8)
    rows, labels, dense = generate_columns(ZipfSpec(schema, 1.05, 40 * 256, seed=5))
    cfg = eng.EngineConfig(cache_capacity=2000, batch_size=256, lookahead=4, num_shards=1, seed=3)
    plain = eng.run_pipeline(cfg, schema, batchify_columns(rows, labels, dense, 256))
    pinned = [b.pin_memory() for b in batchify_columns(rows, labels, dense, 256)]
    assert sorted(set(int(w) for b in pinned for w in b._memo["pinned_planes"][2])) == [1, 2, 4]
    rep = eng.run_pipeline(cfg, schema, pinned)
    assert rep.to_json_bytes() == plain.to_json_bytes()
    assert rep.final_store_digest == plain.final_store_digest
