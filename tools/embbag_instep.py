"""EmbeddingBag forward / backward inside the DLRM step at Criteo-Kaggle
shape: per-step stage spans (engine CUDA events) of the gather (forward)
and of the backward + optimizer, min / median / mean over the steps, with the
bench's settings (bf16 MLP graph, per-iteration L2 flush overlapped, early
enqueue of the next step).

  python tools/embbag_instep.py [--steps 30]

Environment knobs of the library apply (BAGPIPE_B200_LINK_GATE,
BAGPIPE_B200_DEBUG_SKIP_LINK, BAGPIPE_B200_BWD_VARIANT, ...).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2202_12429_b200 import _lib as L  # noqa: E402
from paper_2202_12429_b200.dlrm import DLRMConfig, DLRMTrainer  # noqa: E402
from paper_2202_12429_b200.engine import EngineConfig, _Pipeline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    sc = bench.schema()
    n = args.warmup + args.steps + 12
    batches = bench.make_batches(n, 1)
    cfg = EngineConfig(cache_capacity=sc.total_rows // 100, batch_size=bench.BATCH, lookahead=0, num_shards=1,
                       seed=11)
    trainer = DLRMTrainer(DLRMConfig(emb_optimizer="sgd", emb_lr=0.01, mlp_lr=0.01, mlp_dtype="bf16"),
                          sc.num_dense, sc.num_tables, sc.emb_dim)
    dev = {}
    for i, b in enumerate(batches):
        k, lab, _ = b.packed_occurrences()
        dev[i] = (torch.from_numpy(k).cuda(), torch.from_numpy(lab).cuda())
        trainer.set_device_dense(i, torch.from_numpy(np.ascontiguousarray(b.dense, dtype=np.float32)).cuda(),
                                 torch.from_numpy(b.labels.astype(np.float32)).cuda())
    pipe = _Pipeline(cfg, sc, batches, None, None, device_inputs=dev, timing=True, trainer=trainer)
    pipe.begin()
    for pos in range(args.warmup):
        pipe.step(pos)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    L.check(pipe.lib.bp_engine_set_l2_flush(pipe.eng, L.ptr(flush), flush.numel(), 0), "flush")
    pipe.lib.bp_engine_set_timing(pipe.eng, 1)
    pipe.stage_times()
    fwd, bwd = [], []
    for i in range(args.steps):
        pipe.step(args.warmup + i, early=False)
        st = pipe.stage_times()
        fwd.append(st["trainer"][0] * 1e3)
        bwd.append(st["trainer_bwd"][0] * 1e3)
    pipe.close()

    def summ(x):
        return {"min": round(min(x), 2), "median": round(statistics.median(x), 2), "mean": round(statistics.mean(x), 2)}

    print(json.dumps({"gather_us": summ(fwd), "scatter_us": summ(bwd),
                      "env": {k: v for k, v in os.environ.items() if k.startswith("BAGPIPE_B200_")}}))


if __name__ == "__main__":
    main()
