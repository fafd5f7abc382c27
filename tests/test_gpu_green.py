"""Green-context SM partition of the engine's host-link streams
(`csrc/green.cu`): sized by the row width when left on auto (in the
driver's 8-SM split granularity), and the run it partitions is
byte-identical to an unpartitioned one.  The partition is
process-wide (made at the first engine), so each case runs in its own
interpreter."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np
from paper_2202_12429_b200 import _lib as L
from paper_2202_12429_b200.engine import EngineConfig, run_pipeline
from paper_2202_12429_b200.traces import Schema, ZipfSpec, batchify_columns, generate_columns

dim = int(sys.argv[1])
schema = Schema(4, (50, 3000, 20000, 7), 1, dim)
rows, labels, dense = generate_columns(ZipfSpec(schema, 1.1, 12 * 512, seed=4))
batches = batchify_columns(rows, labels, None, 512)
cfg = EngineConfig(cache_capacity=2000, batch_size=512, lookahead=0, num_trainers=2, num_shards=2, seed=3)
pipe = run_pipeline(cfg, schema, batches)
info = np.zeros(2, dtype=np.int32)
L.check(L.lib().bp_green_info(info.ctypes.data), "bp_green_info")
print(json.dumps({"hot": int(info[0]), "rest": int(info[1]), "digest": pipe.final_store_digest}))
"""


def _run(dim: int, green_sms: str | None) -> dict:
    env = dict(os.environ)
    env.pop("BAGPIPE_B200_GREEN_SMS", None)
    if green_sms is not None:
        env["BAGPIPE_B200_GREEN_SMS"] = green_sms
    out = subprocess.run([sys.executable, "-c", CHILD, str(dim)], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("dim,want_hot", [(16, 8), (64, 16)])
def test_auto_partition_by_row_width_byte_identical(dim, want_hot):
    auto = _run(dim, None)
    assert auto["hot"] == want_hot
    assert auto["rest"] > 100
    off = _run(dim, "0")
    assert off["hot"] == 0 and off["rest"] == 0
    assert auto["digest"] == off["digest"]
