"""Host report format and engine config validation (no GPU)."""

from __future__ import annotations

import json

import pytest

from conftest import golden
from paper_2202_12429_b200.errors import ConfigurationError, TraceFormatError
from paper_2202_12429_b200.report import CSV_COLUMNS, IterationRecord, RunReport, load_report


def test_report_round_trip_matches_reference_bytes(tmp_path):
    blob = golden("reports_small.json")["L8_T1"]
    data = json.loads(blob["json"])
    path = tmp_path / "r.json"
    path.write_text(blob["json"])
    rep = load_report(str(path))
    assert rep.to_json_bytes().decode() == blob["json"]
    header = blob["csv"].split("\n")[0]
    assert header == ",".join(CSV_COLUMNS)
    assert rep.final_store_digest == data["final_store_digest"]


def test_csv_row_format():
    r = IterationRecord(3, True, 1.0, 0.05, 0.25, 0.0, 0.1, 7, 5, 9, 4, 5, 50, 25, 8)
    assert r.csv_row() == "3,1,1.0,0.05,0.25,0.0,0.1,7,5,9,4,5,50,25,8"


def test_load_report_missing_field(tmp_path):
    path = tmp_path / "bad.json"
    path.write_text(json.dumps({"kind": "x"}))
    with pytest.raises(TraceFormatError):
        load_report(str(path))


@pytest.mark.parametrize("bad", [dict(cache_capacity=0), dict(batch_size=0), dict(lookahead=-1),
                                 dict(num_trainers=0), dict(rpc_batch_proportion=0.0),
                                 dict(rpc_batch_proportion=1.5), dict(sync_bandwidth=0.0), dict(mode="parallel")])
def test_config_validation(bad):
    from paper_2202_12429_b200.engine import EngineConfig

    fields = dict(cache_capacity=10, batch_size=2)
    fields.update(bad)
    with pytest.raises(ConfigurationError):
        EngineConfig(**fields)


def test_config_dict_round_trip():
    from paper_2202_12429_b200.engine import EngineConfig

    cfg = EngineConfig(cache_capacity=10, batch_size=2, lookahead=3, mode="threaded")
    assert EngineConfig.from_dict(cfg.to_dict()) == cfg
    with pytest.raises(ConfigurationError):
        EngineConfig.from_dict({"cache_capacity": 5, "batch_size": 2, "bogus": 1})
