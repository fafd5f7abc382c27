"""Isolated timing of the fused DLRM interaction kernels at the Criteo-Kaggle
DLRM-step shape (B = 16,384, T = 26, D = 16, bf16 dense side, gradients stored
in a permuted row order as in the step): CUDA events around each call, L2
flushed before each, median of R.

  python tools/ix_bench.py [--reps 30]

prints one JSON line {kernel: median us}.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2202_12429_b200 import _lib as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--lib", default=None, help="time another build of the library (A/B)")
    args = ap.parse_args()
    lib = L.lib() if args.lib is None else L.load_library(args.lib)
    B, T, D = 16384, 26, 16
    n = T + 1
    P = n * (n - 1) // 2
    out_stride = (D + P + 7) // 8 * 8
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(B, D, device="cuda", generator=g).to(torch.bfloat16)
    emb = torch.randn(B, T, D, device="cuda", generator=g)
    out = torch.empty(B, out_stride, device="cuda", dtype=torch.bfloat16)
    gout = torch.randn(B, out_stride, device="cuda", generator=g).to(torch.bfloat16)
    rows = torch.randperm(B * T, device="cuda", generator=g).to(torch.int32)
    gx = torch.empty_like(x)
    gemb = torch.empty_like(emb)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = L.stream_ptr()

    def fwd():
        L.check(lib.bp_dlrm_interact_forward(L.ptr(x), 1, L.ptr(emb), B, T, D, L.ptr(out), 1, out_stride, s),
                "bp_dlrm_interact_forward")

    def bwd():
        L.check(lib.bp_dlrm_interact_backward_rows(L.ptr(x), 1, L.ptr(emb), L.ptr(gout), 1, B, T, D, out_stride,
                                                   L.ptr(gx), L.ptr(gemb), L.ptr(rows), s),
                "bp_dlrm_interact_backward_rows")

    res = {}
    for name, fn in (("interact_fwd", fwd), ("interact_bwd_rows", bwd)):
        for _ in range(3):
            fn()
        times = []
        for _ in range(args.reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            times.append(a.elapsed_time(b) * 1e3)
        res[name] = float(np.median(times))
    # checksum of the backward outputs (same inputs -> same bits across builds)
    res["fwd_checksum"] = float(out.double().sum())
    res["bwd_checksum"] = [float(gx.float().sum()), float(gemb.double().sum())]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
