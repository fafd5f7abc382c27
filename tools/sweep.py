"""BASELINE.json configs[4]: lookahead window x cache size x Zipf skew at the
Criteo-Kaggle shape, B200 engine vs the CPU oracle of the reference pipeline.

  python tools/sweep.py [--batches 12] [--windows 50,200,1000] [--caches 0.1,1,5] [--zipfs 0.8,1.05,1.2]

Per cell (independent runs, one GPU each): the pipelined engine
(run_pipeline) and the oracle pipeline (oracle/, the reference algorithm)
on the same trace.  Outcome must agree: both finish -- then every written
store row is compared bit for bit -- or both raise the capacity error at the
same iteration (reference cache.py:113-116: literal L=200 at 1% of rows
overflows at iteration 11).  Prints one JSON object with a row
per cell: outcome on both sides, final lookahead, B200 wall ms per
iteration (measured-timing sidecar) and the oracle's CPU ms per iteration.
"""

from __future__ import annotations

import argparse
import json
import os
import re
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=12)
    ap.add_argument("--windows", default="50,200,1000")
    ap.add_argument("--caches", default="0.1,1,5")
    ap.add_argument("--zipfs", default="0.8,1.05,1.2")
    args = ap.parse_args()
    import torch

    from oracle import bagpipe_oracle as O
    from paper_2202_12429_b200.engine import EngineConfig, run_pipeline
    from paper_2202_12429_b200.errors import CacheCapacityError
    from paper_2202_12429_b200.traces import ZipfSpec, batchify_columns, generate_columns

    sc = bench.schema()
    cells = []
    for zipf in [float(z) for z in args.zipfs.split(",")]:
        rows, labels, dense = generate_columns(ZipfSpec(sc, zipf, args.batches * bench.BATCH, 1))
        batches = batchify_columns(rows, labels, dense, bench.BATCH)
        for pct in [float(c) for c in args.caches.split(",")]:
            cap = max(1, int(sc.total_rows * pct / 100))
            for window in [int(w) for w in args.windows.split(",")]:
                cell = {"zipf": zipf, "cache_pct": pct, "capacity": cap, "window": window}
                cfg = EngineConfig(cache_capacity=cap, batch_size=bench.BATCH, lookahead=window, num_shards=1,
                                   seed=11)
                t0 = time.perf_counter()
                try:
                    rep = run_pipeline(cfg, sc, batches, measure_stages=False)
                    wall = rep.measured["wall_ms_per_iteration"]
                    cell["b200"] = {"outcome": "ok", "final_lookahead": rep.final_lookahead,
                                    "ms_per_iteration": float(np.median(wall)) if wall else None}
                    got = {(k[0] << 44) | k[1]: v for k, v in rep.final_store.written_items()}
                    del rep
                except CacheCapacityError as err:
                    it = int(re.search(r"iteration (\d+)", str(err)).group(1))
                    cell["b200"] = {"outcome": f"CacheCapacityError at iteration {it}"}
                    got = None
                cell["b200"]["wall_s"] = round(time.perf_counter() - t0, 2)
                torch.cuda.empty_cache()
                t0 = time.perf_counter()
                try:
                    want, _ = O.pipeline(batches, sc.rows_per_table, sc.emb_dim, 11, 1, cap, window, 0.25)
                    cell["oracle"] = {"outcome": "ok"}
                except RuntimeError as err:
                    it = int(re.search(r"at (\d+)", str(err)).group(1))
                    cell["oracle"] = {"outcome": f"CacheCapacityError at iteration {it}"}
                    want = None
                dt = time.perf_counter() - t0
                cell["oracle"]["ms_per_iteration"] = round(dt * 1e3 / args.batches, 1)
                cell["same_outcome"] = cell["b200"]["outcome"] == cell["oracle"]["outcome"]
                if got is not None and want is not None:
                    same = set(got) == set(want.values) and all(np.array_equal(got[k], v)
                                                                for k, v in want.values.items())
                    cell["written_rows"] = len(got)
                    cell["rows_bit_exact"] = bool(same)
                cells.append(cell)
                print(json.dumps(cell), file=sys.stderr, flush=True)
    print(json.dumps({"config": "BASELINE configs[4] sweep at Criteo-Kaggle shape", "batches": args.batches,
                      "batch": bench.BATCH, "cells": cells,
                      "all_agree": all(c["same_outcome"] and c.get("rows_bit_exact", True) for c in cells)}))


if __name__ == "__main__":
    main()
