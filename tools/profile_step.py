"""Profile engine steps at the Criteo-Kaggle bench shape.

  python tools/profile_step.py [--steps 3] [--nvtx] [--torch-prof]

--nvtx wraps each profiled step in an NVTX range "timed_step" so that
  ncu --nvtx --nvtx-include "timed_step/" ... captures only those launches.
--torch-prof prints a per-kernel device-time table (torch profiler / CUPTI).
"""

from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2202_12429_b200.engine import EngineConfig, _Pipeline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--nvtx", action="store_true")
    ap.add_argument("--torch-prof", action="store_true")
    ap.add_argument("--host-inputs", action="store_true")
    ap.add_argument("--pin", action="store_true", help="host inputs in pinned memory (bench.py's e2e)")
    ap.add_argument("--cprofile", action="store_true")
    ap.add_argument("--trace", default=None, help="write a chrome trace (kernel timeline per stream) here")
    ap.add_argument("--flush", action="store_true", help="256 MiB L2 flush before each step, like bench.py")
    ap.add_argument("--sync-flush", action="store_true", help="drain all engine streams before each flush")
    ap.add_argument("--engine-flush", type=int, default=-1,
                    help="flush inside the engine at each iteration start (0: overlapped, 1: exclusive)")
    ap.add_argument("--link-blocks", type=int, default=0, help="grid of the host-link kernels (0: default)")
    ap.add_argument("--link-config", default="", help="blocks,threads,smem of the host-link kernels")
    ap.add_argument("--skip-link", type=int, default=0,
                    help="debug: 1 = no fetch kernels, 2 = no write-back kernels, 3 = neither (wrong results)")
    ap.add_argument("--dlrm", action="store_true", help="DLRM mode (EmbeddingBag + MLP graph) instead of the stub")
    args = ap.parse_args()
    if args.skip_link:
        from paper_2202_12429_b200 import _lib as L

        L.check(L.lib().bp_debug_skip_link(args.skip_link), "bp_debug_skip_link")
    if args.link_config:
        from paper_2202_12429_b200 import _lib as L

        L.check(L.lib().bp_set_link_config(*[int(x) for x in args.link_config.split(",")]), "bp_set_link_config")
    if args.link_blocks:
        from paper_2202_12429_b200 import _lib as L

        L.check(L.lib().bp_set_link_blocks(args.link_blocks), "bp_set_link_blocks")
    sc = bench.schema()
    n = args.warmup + args.steps + 12
    batches = bench.make_batches(n, 1)
    cfg = EngineConfig(cache_capacity=sc.total_rows // 100, batch_size=bench.BATCH, lookahead=0, num_shards=1,
                       seed=11)
    dev = None
    if args.host_inputs and args.pin:
        for b in batches:
            b.pin_memory()
    if not args.host_inputs:
        dev = {}
        for i, b in enumerate(batches):
            k, lab, _ = b.packed_occurrences()
            dev[i] = (torch.from_numpy(k).cuda(), torch.from_numpy(lab).cuda())
    trainer = None
    if args.dlrm:
        from paper_2202_12429_b200.dlrm import DLRMConfig, DLRMTrainer

        trainer = DLRMTrainer(DLRMConfig(mlp_dtype="bf16"), sc.num_dense, sc.num_tables, sc.emb_dim)
        for i, b in enumerate(batches):
            trainer.set_device_dense(i, torch.from_numpy(b.dense.astype("float32")).cuda(),
                                     torch.from_numpy(b.labels.astype("float32")).cuda())
    pipe = _Pipeline(cfg, sc, batches, None, None, device_inputs=dev, trainer=trainer)
    pipe.begin()
    for pos in range(args.warmup):
        pipe.step(pos)
    torch.cuda.synchronize()
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if args.flush else None

    if args.engine_flush >= 0:
        from paper_2202_12429_b200 import _lib as L

        flush_buf = None
        eng_flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        L.check(pipe.lib.bp_engine_set_l2_flush(pipe.eng, L.ptr(eng_flush), eng_flush.numel(), args.engine_flush),
                "bp_engine_set_l2_flush")

    def one(i):
        if flush_buf is not None and args.sync_flush:
            pipe.lib.bp_engine_sync(pipe.eng)
        if flush_buf is not None:
            with torch.cuda.stream(pipe.stream):
                flush_buf.zero_()
        pipe.step(args.warmup + i)

    if args.torch_prof or args.trace:
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            for i in range(args.steps):
                one(i)
            torch.cuda.synchronize()
        if args.trace:
            prof.export_chrome_trace(args.trace)
            return
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=40))
        print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
        return
    if args.cprofile:
        import cProfile
        import pstats

        pr = cProfile.Profile()
        pr.enable()
        for i in range(args.steps):
            pipe.step(args.warmup + i)
        torch.cuda.synchronize()
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(30)
        return
    t0 = time.perf_counter()
    for i in range(args.steps):
        if args.nvtx:
            torch.cuda.nvtx.range_push("timed_step")
        one(i)
        if args.nvtx:
            torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    print(f"{args.steps} steps in {(time.perf_counter() - t0) * 1e3:.2f} ms")
    import numpy as np

    from paper_2202_12429_b200 import _lib as L

    st = np.zeros(9, dtype=np.int64)
    L.lib().bp_debug_link_cb_stats(st.ctypes.data)
    print(f"host workers: gather {st[1]} calls {st[2]} rows {st[0] / 1e3:.0f} us; "
          f"scatter {st[4]} calls {st[5]} rows {st[3] / 1e3:.0f} us; upload copies {st[7]} calls "
          f"{st[8] / 1e6:.1f} MB {st[6] / 1e3:.0f} us")


if __name__ == "__main__":
    main()
