"""Host-side cost of the engine's iteration loop (stub mode, CK shape, N=1):
cProfile over K bench-style steps with device-resident batches, top
functions by own time, plus the per-step host time outside the waits.

  python tools/host_profile.py [--steps 200] [--top 30]
"""

from __future__ import annotations

import argparse
import cProfile
import io
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--top", type=int, default=30)
    args = ap.parse_args()
    import torch

    from paper_2202_12429_b200.engine import EngineConfig, _Pipeline

    sc = bench.schema()
    warm = 5
    batches = bench.make_batches(warm + args.steps + 10, 1)
    cap = max(1, int(sc.total_rows * 0.01))
    cfg = EngineConfig(cache_capacity=cap, batch_size=bench.BATCH, lookahead=0, num_trainers=1, num_shards=1,
                       seed=11)
    dev = {}
    for i, b in enumerate(batches):
        keys, labels, _ = b.packed_occurrences()
        dev[i] = (torch.from_numpy(keys).cuda(), torch.from_numpy(labels).cuda())
    torch.cuda.synchronize()
    pipe = _Pipeline(cfg, sc, batches, None, None, device_inputs=dev)
    pipe.begin()
    for pos in range(warm):
        pipe.step(pos)
    torch.cuda.synchronize()
    # plain pass first: host busy time per step without the profiler
    half = args.steps // 2
    w0, t0 = pipe.host_wait_s, time.perf_counter()
    for i in range(half):
        pipe.step(warm + i)
    torch.cuda.synchronize()
    wall0, wait0 = time.perf_counter() - t0, pipe.host_wait_s - w0
    print(f"plain: wall {wall0 * 1e6 / half:.1f} us/step, host wait {wait0 * 1e6 / half:.1f}, "
          f"host busy {(wall0 - wait0) * 1e6 / half:.1f} us/step", flush=True)
    warm += half
    args.steps -= half
    prof = cProfile.Profile()
    w0 = pipe.host_wait_s
    t0 = time.perf_counter()
    prof.enable()
    for i in range(args.steps):
        pipe.step(warm + i, early=i < args.steps - 1)
    prof.disable()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    wait = pipe.host_wait_s - w0
    out = io.StringIO()
    pstats.Stats(prof, stream=out).sort_stats("tottime").print_stats(args.top)
    print(out.getvalue())
    print(f"cProfile: wall {wall * 1e6 / args.steps:.1f} us/step, host wait {wait * 1e6 / args.steps:.1f} "
          f"us/step, host busy {(wall - wait) * 1e6 / args.steps:.1f} us/step")


if __name__ == "__main__":
    main()
