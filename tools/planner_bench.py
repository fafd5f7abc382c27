"""Batch prep + Oracle Cacher planner at Criteo-Kaggle shape, isolated.

  python tools/planner_bench.py [--batches 24] [--lookahead 7] [--nvtx]

Runs the planner's steady state the way the engine does (one prep per batch
entering the window, refill with it, pop the window's front batch) on one
stream, device-resident keys, and prints one JSON line:

* prep_us / planner_us: CUDA-event time per batch of bp_prep_create_columnar
  and of refill + pop, averaged over the steady-state batches;
* kernels_us: per-kernel device time per batch (CUPTI, torch profiler);
* algorithmic bytes per batch and the GB/s they imply:
    prep:    keys + labels read (9 B/occ), sorted positions + label bytes
             written (5 B/occ), per unique key: sorted key, id, first-order
             key, both permutations, CSR offset (32 B)
    planner: refill ids read + tracker/flag write (13 B/unique), pop ids /
             tracker / flags read + ttl + flags written (21 B/unique),
             prefetch key/id/ttl (20 B), evict key/id (12 B).
--nvtx wraps the steady-state batches in an NVTX range "planner_batch" for
  ncu --nvtx --nvtx-include "planner_batch/".
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2202_12429_b200 import _lib as L  # noqa: E402
from paper_2202_12429_b200.device import DevicePrep, DeviceSchema  # noqa: E402


def prep_bytes(n_occ: int, u: int) -> int:
    return n_occ * (9 + 5) + u * 32


def planner_bytes(u: int, p: int, e: int) -> int:
    return u * (13 + 21) + p * 20 + e * 12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=24)
    ap.add_argument("--lookahead", type=int, default=7)
    ap.add_argument("--warm", type=int, default=10)
    ap.add_argument("--nvtx", action="store_true")
    ap.add_argument("--no-prof", action="store_true")
    ap.add_argument("--trace", action="store_true", help="phase timestamps of the cluster prep and the fused pop")
    args = ap.parse_args()
    lib = L.lib()
    sc = bench.schema()
    batches = bench.make_batches(args.batches + args.lookahead, 1)
    ds = DeviceSchema.get(sc)
    cap = sc.total_rows // 100
    stream = torch.cuda.Stream()
    dev = []
    for b in batches:
        k, lab, _ = b.packed_occurrences()
        dev.append((k, lab, torch.from_numpy(k).cuda(), torch.from_numpy(lab).cuda(),
                    (b.num_examples, b.table_ids()), b.rank_bounds(1), b.iteration))
    torch.cuda.synchronize()
    h = C.c_void_p()
    L.check(lib.bp_planner_create(L.Context.get().handle, ds.handle, cap, C.byref(h)), "bp_planner_create")
    n_occ = len(dev[0][0])
    bufs = dict(keys=torch.empty(n_occ, dtype=torch.uint64, device="cuda"),
                ids=torch.empty(n_occ, dtype=torch.uint32, device="cuda"),
                ttls=torch.empty(n_occ, dtype=torch.int64, device="cuda"),
                ttl_k=torch.empty(n_occ, dtype=torch.int64, device="cuda"),
                ev=torch.empty(n_occ, dtype=torch.uint64, device="cuda"),
                ev_ids=torch.empty(n_occ, dtype=torch.uint32, device="cuda"),
                counts=torch.zeros(5, dtype=torch.int64, device="cuda"))
    pb = L.PlanBuffers(*(L.ptr(bufs[k]) for k in ("keys", "ids", "ttls", "ttl_k", "ev", "ev_ids", "counts")))
    preps = {}

    def make(i):
        k, lab, dk, dl, cols, rb, it = dev[i]
        return DevicePrep(k, lab, rb, it, sc, 0, stream, d_keys=dk, d_labels=dl, columns=cols)

    sp = L.stream_ptr(stream)
    Lw = args.lookahead
    for j in range(Lw - 1):
        preps[j] = make(j)
        L.check(lib.bp_planner_refill(h, preps[j].handle, sp), "refill")
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t_prep, t_plan, us, pfs, evs = [], [], [], [], []

    def one(i, timed):
        j = i + Lw - 1
        a, b, c = ev(), ev(), ev()
        a.record(stream)
        preps[j] = make(j)
        b.record(stream)
        L.check(lib.bp_planner_refill(h, preps[j].handle, sp), "refill")
        L.check(lib.bp_planner_pop(h, preps[i].handle, C.byref(pb), sp), "pop")
        c.record(stream)
        stream.synchronize()
        if timed:
            t_prep.append(a.elapsed_time(b) * 1e3)
            t_plan.append(b.elapsed_time(c) * 1e3)
            cnt = bufs["counts"].cpu().numpy()
            pfs.append(int(cnt[0]))
            evs.append(int(cnt[1]))
            us.append(preps[i].num_unique)
        preps.pop(i).destroy()

    i = 0
    for _ in range(args.warm):
        one(i, False)
        i += 1
    n_timed = args.batches - args.warm - 2
    for _ in range(n_timed):
        if args.nvtx:
            torch.cuda.nvtx.range_push("planner_batch")
        one(i, True)
        if args.nvtx:
            torch.cuda.nvtx.range_pop()
        i += 1
    kernels = {}
    if not args.no_prof:
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            one(i, False)
            torch.cuda.synchronize()
        i += 1
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CUDA:
                name = (e.name or "").split("(")[0].replace("void ", "")
                kernels[name] = round(kernels.get(name, 0.0) + e.device_time, 2)
    trace = None
    if args.trace:
        tp = torch.zeros(64 * 16 * 16, dtype=torch.int64, device="cuda")
        tq = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
        L.check(lib.bp_debug_phase_trace(0, L.ptr(tp)), "trace")
        L.check(lib.bp_debug_phase_trace(1, L.ptr(tq)), "trace")
        one(i, False)
        i += 1
        L.check(lib.bp_debug_phase_trace(0, None), "trace")
        L.check(lib.bp_debug_phase_trace(1, None), "trace")
        a = tp.view(64, 16, 16).cpu().numpy()
        ncols = len(dev[0][4][1])
        a = a[:ncols]
        valid = a[:, :, 0] > 0
        t0 = a[:, :, 0][valid].min()
        cols = {}
        for c in range(ncols):
            v = a[c][valid[c]]
            rel = np.where(v > 0, (v - t0) / 1e3, np.nan)
            cols[c] = {"ctas": int(valid[c].sum()), "max_us": [None if np.isnan(x) else round(float(x), 2)
                                                               for x in np.nanmax(rel, axis=0)[:11]],
                       "min_us": [None if np.isnan(x) else round(float(x), 2) for x in np.nanmin(rel, axis=0)[:11]]}
        q = tq.view(4096, 8).cpu().numpy()
        qv = q[q[:, 0] > 0]
        q0 = qv[:, 0].min()
        qrel = (qv[:, :5] - q0) / 1e3
        trace = {"prep_phases": "0 start, 1 loads, 2-5 after radix pass 1-4, 6 final sync, 7 heads counted, "
                                "8 column look-back, 9 outputs, 10 long list",
                 "prep_columns": cols,
                 "pop_phases": "0 start, 1 loads+decisions, 2 block scan, 3 look-back, 4 compaction",
                 "pop_tiles": int(len(qv)), "pop_max_us": [round(float(x), 2) for x in qrel.max(axis=0)],
                 "pop_min_us": [round(float(x), 2) for x in qrel.min(axis=0)],
                 "pop_median_us": [round(float(x), 2) for x in np.median(qrel, axis=0)]}
    u, p, e = float(np.mean(us)), float(np.mean(pfs)), float(np.mean(evs))
    prep_us, plan_us = float(np.median(t_prep)), float(np.median(t_plan))
    pb_, plb = prep_bytes(n_occ, int(u)), planner_bytes(int(u), int(p), int(e))
    out = {"n_occ": n_occ, "unique": u, "prefetch": p, "evict": e, "lookahead": Lw,
           "prep_us": prep_us, "planner_us": plan_us, "prep_plus_planner_us": prep_us + plan_us,
           "prep_bytes": pb_, "planner_bytes": plb,
           "prep_gbs": pb_ / (prep_us * 1e-6) / 1e9, "planner_gbs": plb / (plan_us * 1e-6) / 1e9,
           "combined_gbs": (pb_ + plb) / ((prep_us + plan_us) * 1e-6) / 1e9,
           "prep_us_all": [round(x, 1) for x in t_prep], "planner_us_all": [round(x, 1) for x in t_plan],
           "kernels_us": kernels, "trace": trace}
    print(json.dumps(out), flush=True)
    lib.bp_planner_destroy(h)


if __name__ == "__main__":
    main()
