"""Isolated timings of the hot kernels on one Criteo-Kaggle batch (no engine,
no host-link traffic competing): CUDA events around R repetitions, L2
flushed before each.

  python tools/kernel_bench.py [--reps 20]

prints one JSON line: per kernel family the mean microseconds per call.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2202_12429_b200 import _lib as L  # noqa: E402
from paper_2202_12429_b200.device import DevicePrep  # noqa: E402


def timed(fn, reps, flush):
    times = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b) * 1e3)
    return float(np.median(times))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    lib = L.lib()
    sc = bench.schema()
    batch = bench.make_batches(1, 1)[0]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {}
    dim = bench.DIM

    # batch prep (columnar per-table sort + segments) from device-resident keys
    keys, labels, _ = batch.packed_occurrences()
    d_keys, d_labels = torch.from_numpy(keys).cuda(), torch.from_numpy(labels).cuda()
    cols = (batch.num_examples, batch.table_ids())
    rb = batch.rank_bounds(1)

    def make_prep(flags=0):
        return DevicePrep(keys, labels, rb, batch.iteration, sc, flags, d_keys=d_keys, d_labels=d_labels,
                          columns=cols)

    prep = make_prep()
    keep = []
    # event span around the whole Python-level DevicePrep construction (host
    # argument marshalling, arena allocation and launches included); the
    # prep kernels' own device time is in kernels_us (k_col_cluster_prep,
    # k_first_order) and in tools/planner_bench.py
    out["prep_construct_span_us"] = timed(lambda: keep.append(make_prep()), args.reps, flush)
    keep.clear()

    u = prep.num_unique
    rows = torch.randn((u, dim), dtype=torch.float32, device="cuda") * 0.05
    row_index = torch.arange(u, dtype=torch.int32, device="cuda")
    dirty = torch.zeros(u, dtype=torch.uint8, device="cuda")
    ctx = L.Context.get().handle

    def stub():
        f = float(np.float32(0.01))
        L.check(lib.bp_stub_step(ctx, prep.handle, L.ptr(rows), L.ptr(row_index), L.ptr(dirty), dim, f,
                                 float(np.float32(0.001)), f, 0, None, None, 0, None, L.stream_ptr()), "bp_stub_step")

    out["stub_step_us"] = timed(stub, args.reps, flush)
    # phase clocks of the long-segment kernel's CTAs (the hottest chain)
    trace = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    L.check(lib.bp_debug_long_trace(L.ptr(trace)), "bp_debug_long_trace")
    flush.zero_()
    stub()
    torch.cuda.synchronize()
    L.check(lib.bp_debug_long_trace(None), "bp_debug_long_trace")
    tr = trace.view(148, 8).cpu().numpy()
    hot = int(np.argmax(tr[:, 5]))
    t = tr[hot]
    out["long_hot_cta"] = {"occurrences": int(t[5]), "setup_cyc": int(t[1] - t[0]), "window_cyc": int(t[2] - t[1]),
                           "chain_cyc": int(t[3] - t[2]), "tail_cyc": int(t[4] - t[3]),
                           "cta_total_cyc": int(t[4] - t[0])}
    starts = tr[:, 0]
    out["long_cta_start_spread_cyc"] = int(starts.max() - starts.min())
    # the same chain with the short-segment kernel serialised after it (no
    # co-resident warps competing for the chain warp's issue slots)
    L.check(lib.bp_set_stub_fork(0), "bp_set_stub_fork")
    trace.zero_()
    L.check(lib.bp_debug_long_trace(L.ptr(trace)), "bp_debug_long_trace")
    flush.zero_()
    stub()
    torch.cuda.synchronize()
    L.check(lib.bp_debug_long_trace(None), "bp_debug_long_trace")
    out["stub_step_serial_us"] = timed(stub, args.reps, flush)
    L.check(lib.bp_set_stub_fork(2), "bp_set_stub_fork")
    t = trace.view(148, 8).cpu().numpy()[hot]
    out["long_hot_cta_alone"] = {"occurrences": int(t[5]), "chain_cyc": int(t[3] - t[2]),
                                 "cyc_per_occurrence": round(float(t[3] - t[2]) / max(int(t[5]), 1), 2)}

    # EmbeddingBag forward / backward (DLRM prep: occurrence->unique maps)
    prep2 = make_prep(2)
    u2 = prep2.num_unique
    values = torch.randn((u2, dim), dtype=torch.float32, device="cuda")
    slots = torch.arange(u2, dtype=torch.int32, device="cuda")
    n = prep2.n_occ
    pooled = torch.empty((n, dim), dtype=torch.float32, device="cuda")
    grad = torch.randn((n, dim), dtype=torch.float32, device="cuda") * 1e-3

    def fwd():
        L.check(lib.bp_embbag_forward(prep2.handle, L.ptr(values), dim, L.ptr(slots), dim, None, n, 0, None,
                                      L.ptr(pooled), L.stream_ptr()), "fwd")

    def bwd():
        L.check(lib.bp_embbag_backward(prep2.handle, L.ptr(grad), None, None, L.ptr(values), dim, L.ptr(slots), None,
                                       dim, 0, float(np.float32(0.01)), 0.0, None, L.stream_ptr()), "bwd")

    def bwd_sorted():  # gradients in key-sorted order (as the interaction backward stores them)
        L.check(lib.bp_embbag_backward_sorted(prep2.handle, L.ptr(grad), L.ptr(values), dim, L.ptr(slots), None,
                                              dim, 0, float(np.float32(0.01)), 0.0, None, L.stream_ptr()),
                "bwd sorted")

    # warm: the gradient rows just written (L2-resident, as after the
    # interaction backward in a DLRM step), no flush
    grad_src = grad.clone()

    def timed_warm(fn, reps):
        times = []
        for _ in range(reps):
            grad.copy_(grad_src)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            times.append(a.elapsed_time(b) * 1e3)
        return float(np.median(times))

    out["embbag_bwd_warm_us"] = timed_warm(bwd, args.reps)
    for var in (0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10):
        lib.bp_debug_bwd_variant(var)
        out[f"embbag_bwd_sorted_v{var}_warm_us"] = timed_warm(bwd_sorted, args.reps)
    lib.bp_debug_bwd_variant(-1)
    out["embbag_fwd_us"] = timed(fwd, args.reps, flush)
    lib.bp_debug_fwd_variant(1)
    out["embbag_fwd_sorted_us"] = timed(fwd, args.reps, flush)
    ref = pooled.clone()
    lib.bp_debug_fwd_variant(0)
    fwd()
    out["embbag_fwd_variants_equal"] = bool(torch.equal(ref, pooled))
    out["embbag_bwd_us"] = timed(bwd, args.reps, flush)
    out["embbag_bwd_sorted_us"] = timed(bwd_sorted, args.reps, flush)
    for var in (0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10):  # launch shapes (0: staged, 4: split, 5: persistent, 6: small staged, 7: no end list, 8/9: register reduce + apply)
        lib.bp_debug_bwd_variant(var)
        out[f"embbag_bwd_sorted_v{var}_us"] = timed(bwd_sorted, args.reps, flush)
    lib.bp_debug_bwd_variant(-1)
    fwd_bytes = n * (8 * dim + 4)
    bwd_bytes = n * (4 * dim + 4) + u2 * (8 * dim)
    out["embbag_fwd_gbs"] = fwd_bytes / (out["embbag_fwd_us"] * 1e-6) / 1e9
    out["embbag_bwd_gbs"] = bwd_bytes / (out["embbag_bwd_us"] * 1e-6) / 1e9
    out["embbag_fwd_bwd_gbs"] = (fwd_bytes + bwd_bytes) / ((out["embbag_fwd_us"] + out["embbag_bwd_us"]) * 1e-6) / 1e9
    out["embbag_bwd_sorted_gbs"] = bwd_bytes / (out["embbag_bwd_sorted_us"] * 1e-6) / 1e9
    out["embbag_fwd_bwd_sorted_gbs"] = (fwd_bytes + bwd_bytes) / (
        (out["embbag_fwd_us"] + out["embbag_bwd_sorted_us"]) * 1e-6) / 1e9
    out["n_occ"], out["unique"] = n, u
    # per-kernel device times (CUPTI) of one call each, L2 flushed first
    from torch.profiler import ProfilerActivity, profile

    kernels = {}

    def variant(v):
        def run():
            lib.bp_debug_bwd_variant(v)
            bwd_sorted()
            lib.bp_debug_bwd_variant(-1)
        return run

    def fwd_sorted():
        lib.bp_debug_fwd_variant(1)
        fwd()
        lib.bp_debug_fwd_variant(0)

    for fn in (lambda: keep.append(make_prep()), stub, fwd, fwd_sorted, bwd, bwd_sorted, variant(0), variant(1), variant(2), variant(3), variant(4), variant(5), variant(6), variant(7), variant(8), variant(10)):  # (variant 9 is the default bwd_sorted)
        flush.zero_()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        for ev in prof.events():
            if ev.device_type == torch.autograd.DeviceType.CUDA and "bp::" in (ev.name or ""):
                name = ev.name.split("(")[0].replace("void ", "")
                kernels[name] = round(kernels.get(name, 0.0) + ev.device_time, 2)
    out["kernels_us"] = kernels
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
