"""The CLI over the B200 engine against the reference CLI's own outputs
(tests/golden/cli.json, made by tests/golden/make_golden.py gen_cli from the
reference's cli.main on the fixtures of reference tests/test_cli.py:22-51):
gen-trace file bytes, plan records (incl. the worked-example golden records
of reference tests/test_cli.py:97-103), run/baseline report JSON + CSV bytes
and store dumps, verify exit codes; plus the device trace ingest (EMTRC1
decoded on the GPU) and the measured-timing sidecar."""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from conftest import golden, make_batch
from paper_2202_12429_b200.cli import main
from paper_2202_12429_b200.traces import Schema, ZipfSpec, generate_synthetic_trace, write_trace

G = golden("cli.json")


def _sha(path) -> str:
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


@pytest.fixture(scope="module")
def trace_file(tmp_path_factory) -> str:
    path = tmp_path_factory.mktemp("traces") / "zipf.trace"
    schema = Schema(2, (600, 400), 2, 4)
    write_trace(str(path), schema, generate_synthetic_trace(ZipfSpec(schema, 1.05, 30 * 64, seed=7)))
    return str(path)


@pytest.fixture(scope="module")
def worked_trace_file(tmp_path_factory) -> str:
    path = tmp_path_factory.mktemp("traces") / "fig.trace"
    batches = [make_batch(1, [3, 9]), make_batch(2, [3, 4]), make_batch(3, [3, 6]), make_batch(4, [1, 6])]
    write_trace(str(path), Schema(1, (10,), 0, 4), [ex for b in batches for ex in b.examples])
    return str(path)


def config_file(tmp_path, **overrides) -> str:
    cfg = dict(cache_capacity=5_000, batch_size=64, lookahead=8, num_trainers=2, seed=5)
    cfg.update(overrides)
    path = tmp_path / "config.json"
    path.write_text(json.dumps(cfg), encoding="utf-8")
    return str(path)


# ------------------------------------------------------------------ CPU
def test_gen_trace_bytes_match_reference(tmp_path, capsys):
    out = str(tmp_path / "gen.trace")
    assert main(["gen-trace", "--schema", "2:300,200:1:4", "--zipf", "1.05", "--examples", "500", "--seed", "3",
                 "--out", out]) == G["gen_trace"]["rc"] == 0
    assert _sha(out) == G["gen_trace"]["sha256"]
    assert capsys.readouterr().out == f"wrote 500 examples to {out}\n"


def test_usage_errors_exit_2(tmp_path):
    with pytest.raises(SystemExit) as err:
        main(["gen-trace", "--schema", "nope", "--zipf", "1.0", "--examples", "10", "--out", str(tmp_path / "x")])
    assert err.value.code == 2
    with pytest.raises(SystemExit) as err:
        main(["frobnicate"])
    assert err.value.code == 2


def test_missing_trace_is_runtime_error(tmp_path):
    assert main(["plan", "--trace", str(tmp_path / "nope.trace"), "--batch-size", "2", "--lookahead", "2",
                 "--capacity", "10", "--out", str(tmp_path / "p.txt")]) == 3


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_plan_worked_example_records(tmp_path, worked_trace_file):
    out = str(tmp_path / "plans.txt")
    assert main(["plan", "--trace", worked_trace_file, "--batch-size", "2", "--lookahead", "2", "--capacity", "100",
                 "--first-iteration", "1", "--out", out]) == 0
    lines = open(out).read().splitlines()
    assert lines == G["plan_worked"]["lines"] == ["iter=1 prefetch=0:3,0:9 ttl=0:3@2,0:9@1",
                                                 "iter=2 prefetch=0:4 ttl=0:3@3,0:4@2",
                                                 "iter=3 prefetch=0:6 ttl=0:3@3,0:6@4",
                                                 "iter=4 prefetch=0:1 ttl=0:1@4,0:6@4"]


@pytest.mark.gpu
def test_plan_zipf_bytes(tmp_path, trace_file):
    out = str(tmp_path / "plans.txt")
    assert main(["plan", "--trace", trace_file, "--batch-size", "64", "--lookahead", "8", "--capacity", "5000",
                 "--out", out]) == 0
    assert _sha(out) == G["plan_zipf"]["sha256"]


@pytest.mark.gpu
def test_run_baseline_verify_flow_matches_reference(tmp_path, trace_file, capsys):
    cfg = config_file(tmp_path)
    reports = {}
    for cmd in ("run", "baseline"):
        rep = str(tmp_path / f"{cmd}.json")
        assert main([cmd, "--config", cfg, "--trace", trace_file, "--report", rep, "--dump-store"]) == 0
        want = G[cmd]
        assert open(rep).read() == want["json"]
        assert open(rep[:-5] + ".csv").read() == want["csv"]
        assert _sha(rep[:-5] + ".store") == want["store_sha256"]
        assert capsys.readouterr().out == want["stdout"]
        reports[cmd] = rep
    assert main(["verify", "--a", reports["run"], "--b", reports["baseline"]]) == G["verify"]["rc"] == 0
    assert capsys.readouterr().out == G["verify"]["stdout"]
    # incomparable runs (different lr): a runtime error, exit 3 (reference cli.py:245-248)
    cfg2 = config_file(tmp_path, lr=0.02)
    other = str(tmp_path / "other.json")
    assert main(["baseline", "--config", cfg2, "--trace", trace_file, "--report", other]) == 0
    assert main(["verify", "--a", reports["run"], "--b", other]) == 3


@pytest.mark.gpu
def test_run_device_ingest_and_timing_sidecar(tmp_path, trace_file):
    """--device-ingest (EMTRC1 decoded on the GPU) gives the same report bytes;
    --timing writes measured wall clock per iteration and device stage times."""
    cfg = config_file(tmp_path)
    rep = str(tmp_path / "dev.json")
    assert main(["run", "--config", cfg, "--trace", trace_file, "--report", rep, "--device-ingest", "--timing"]) == 0
    assert open(rep).read() == G["run"]["json"]
    assert open(rep[:-5] + ".csv").read() == G["run"]["csv"]
    t = json.load(open(rep[:-5] + ".timing.json"))
    assert len(t["wall_ms_per_iteration"]) == 30 and all(w >= 0 for w in t["wall_ms_per_iteration"])
    assert set(t["stage_ms"]) >= {"prep", "planner", "fetch", "apply", "trainer", "evict", "flush"}
    assert t["ingest"]["records"] == 30 * 64 and t["ingest"]["ingest_gbs"] > 0
    rows = open(rep[:-5] + ".timing.csv").read().splitlines()
    assert rows[0] == "iteration,simulated_time,wall_ms" and len(rows) == 31


@pytest.mark.gpu
def test_device_ingest_decodes_like_the_host_reader(tmp_path):
    """bp_trace_decode == the host EMTRC1 reader (reference traces.py:231-296)
    on a Criteo-Kaggle-shaped trace with a small chunk size (many chunks,
    ragged last chunk)."""
    import torch

    from paper_2202_12429_b200.ingest import read_trace_device
    from paper_2202_12429_b200.traces import generate_columns, pack_keys, read_trace_columns, write_trace_columns

    schema = Schema(26, tuple(range(3, 3 + 26 * 997, 997)), 13, 16)
    rows, labels, dense = generate_columns(ZipfSpec(schema, 1.05, 5000, seed=4))
    path = str(tmp_path / "ck.trace")
    write_trace_columns(path, schema, rows, labels, dense)
    sc, r2, l2, d2 = read_trace_columns(path)
    tr = read_trace_device(path, chunk_bytes=261 * 777)
    assert tr.stats["chunks"] == (5000 + 776) // 777
    t = np.arange(26, dtype=np.int64)
    want = pack_keys(np.broadcast_to(t, r2.shape).reshape(-1), r2.reshape(-1))
    assert np.array_equal(tr.keys.cpu().numpy().view(np.uint64), want)
    assert np.array_equal(tr.labels.cpu().numpy(), l2)
    assert np.array_equal(tr.occ_labels.cpu().numpy(), np.repeat(l2, 26))
    assert np.array_equal(tr.dense.cpu().numpy(), d2)
    ins = tr.batch_inputs(1024)
    assert len(ins) == 5 and ins[4][0].numel() == (5000 - 4096) * 26
    assert isinstance(ins[0][0], torch.Tensor)
