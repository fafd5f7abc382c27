#!/usr/bin/env python
"""Benchmark of the B200 BagPipe embedding-access hot path (one JSON line).

Workload (BASELINE.json configs[1]): Criteo-Kaggle shape -- 26 tables with
the public Kaggle cardinalities (33,762,577 rows), emb dim 16 fp32, batch
16,384, Zipf 1.05 synthetic IDs (reference generator stream), HBM cache = 1%
of rows (337,625 entries), lookahead auto (-> 7), host-pinned embedding
table.  One step = one engine iteration over one batch: plan emission
(GPU dedupe + Algorithm 1), prefetch from the pinned store (written rows over
the host link, never-written rows computed on the GPU), cache insert + TTL +
lookup, fused stub backward + rank-ordered combine + SGD, eviction, batched
dirty write-back (copy-engine log appends) -- the reference's run_pipeline
iteration (engine.py:495-606), bit-exact with it.

value: samples/s with every batch's keys already in HBM; e2e: the same steps
through the public API with host batches in pinned memory (H2D DMA of the
batch entering the window and D2H of the step counters inside the timed
region).  L2 is flushed (256 MiB write on the compute stream) at the start of
every timed iteration.  ``--impl reference`` times the CPU oracle port of the
reference (oracle/, the reference itself is unavailable on the box) on the
host cores.  N>1 (weak scaling, fixed 16,384 examples per GPU): the global
batch is N x 16,384, the N GPUs are the reference's N trainers, and the 26
tables are sharded table-wise over the ranks (each rank runs the whole
pipeline for its tables of every example -- the same occurrences per GPU as
one GPU -- no data-path collective), timed as the max over ranks.
DLRM mode (N=1, reported under "dlrm" and in "roofline"): the same engine
with EmbeddingBag fwd/bwd + SGD feeding PyTorch MLPs replayed as a CUDA graph.
"""

from __future__ import annotations

import argparse
import gc
import json

import numpy as np
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CK_ROWS = (1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683, 8351593, 3194, 27, 14992, 5461306,
           10, 5652, 2173, 4, 7046547, 18, 15, 286181, 105, 142572)
BATCH = 16384
DIM = 16
ZIPF = 1.05
METRIC = "DLRM samples/sec at 1/2/4/8 B200; embedding gather GB/s vs HBM peak"
WORKLOAD = ("criteo-kaggle-shape 26 tables 33.76M rows D=16 fp32, batch 16384, zipf 1.05, HBM cache 1% of rows, "
            "lookahead auto(7), pinned-host table; stub-gradient engine iteration (reference run_pipeline)")


NUM_DENSE = 13
SHAPE = "ck"

# BASELINE.json configs 3 and 4 as alternative workloads (--shape): the
# headline line (the driver's) is configs[1], the Criteo-Kaggle shape.
# Avazu: 22 categorical tables summing to 9,449,206 rows ("9.4M"; the
# split is ours, the reference ships none), D=16, batch 16,384.  tb10: the
# Criteo-Terabyte cardinalities / 10 (88.3M rows, 22.6 GB pinned fp32 store),
# D=64, batch 65,536.
SHAPES = {
    "ck": dict(rows=CK_ROWS, batch=16384, dim=16, dense=13, workload=WORKLOAD),
    "avazu": dict(rows=(7, 7, 4737, 7745, 26, 8552, 559, 36, 2686408, 6729486, 8251, 5, 4, 2626, 8, 9, 435, 4, 68,
                        172, 60, 1), batch=16384, dim=16, dense=1,
                  workload="avazu-shape 22 tables 9.45M rows D=16 fp32, batch 16384, zipf 1.05, HBM cache 1% of "
                           "rows, lookahead auto, pinned-host table; stub-gradient engine iteration"),
    "tb10": dict(rows=tuple(max(1, r // 10) for r in (227605432, 39060, 17295, 7424, 20265, 3, 7122, 1543, 63,
                                                       130229467, 3067956, 405282, 10, 2209, 11938, 155, 4, 976, 14,
                                                       292775614, 40790948, 187188510, 590152, 12973, 108, 36)),
                 batch=65536, dim=64, dense=13,
                 workload="criteo-terabyte-shape / 10: 26 tables 88.3M rows D=64 fp32, batch 65536, zipf 1.05, HBM "
                          "cache 1% of rows, lookahead auto, pinned-host table; stub-gradient engine iteration"),
}


def apply_shape(name: str) -> None:
    """Rebind the workload constants to one of SHAPES."""
    global CK_ROWS, BATCH, DIM, NUM_DENSE, WORKLOAD, SHAPE
    sh = SHAPES[name]
    CK_ROWS, BATCH, DIM, NUM_DENSE, WORKLOAD, SHAPE = (sh["rows"], sh["batch"], sh["dim"], sh["dense"],
                                                       sh["workload"], name)


# N>1 stub-mode sharding: "row" (keys placed by fnv1a64(table, row) mod N,
# the reference store's placement), "table" (whole tables per rank), or
# "auto": tables up to N=4 (measured faster: 0.226 vs 0.281 ms/step at N=4,
# the columnar cluster prep applies), rows from N=8 (26 tables cannot be
# balanced over 8 ranks when one holds 10.1M rows)
SHARDING_MODE = os.environ.get("BAGPIPE_B200_SHARDING", "auto")


def sharding(world: int) -> str:
    if SHARDING_MODE != "auto":
        return SHARDING_MODE
    return "table" if world <= 4 else "row"

# L2 flush at every iteration start: 0 = the memset runs on the compute
# stream while the plan / host-link streams keep working (the pipeline stays
# overlapped across iterations), 1 = every engine stream drained around it
FLUSH_EXCLUSIVE = int(os.environ.get("BAGPIPE_B200_BENCH_FLUSH_EXCLUSIVE", "0"))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-steps", type=int, default=8, help="oracle steps timed for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dlrm", action="store_true")
    ap.add_argument("--no-link-probe", action="store_true", help="skip the host-link-disabled comparison run")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--shape", default="ck", choices=sorted(SHAPES),
                    help="workload: ck (BASELINE configs[1], the headline), avazu (configs[2]), tb10 (configs[3] / 10)")
    return ap.parse_args()


def schema():
    from paper_2202_12429_b200.traces import Schema

    return Schema(len(CK_ROWS), CK_ROWS, NUM_DENSE, DIM)


def make_batches(n_batches: int, seed: int, batch: int = BATCH):
    from paper_2202_12429_b200.traces import ZipfSpec, batchify_columns, generate_columns

    rows, labels, dense = generate_columns(ZipfSpec(schema(), ZIPF, n_batches * batch, seed))
    return batchify_columns(rows, labels, dense, batch)


def make_batches_shared(n_batches: int, seed: int, batch: int, rank: int, world: int):
    """make_batches, generated once per box at N > 1: rank 0 writes the trace
    columns to /dev/shm, the other ranks map them (instead of N processes
    each drawing the whole global trace on the same host cores)."""
    if world == 1:
        return make_batches(n_batches, seed, batch)
    import numpy as np
    import torch.distributed as dist

    from paper_2202_12429_b200.traces import ZipfSpec, batchify_columns, generate_columns

    tag = f"/dev/shm/bp_bench_{os.environ.get('MASTER_PORT', '0')}_{seed}_{n_batches}_{batch}"
    names = ("rows", "labels", "dense")
    ok = [True]
    if rank == 0:
        cols = generate_columns(ZipfSpec(schema(), ZIPF, n_batches * batch, seed))
        try:
            for name, arr in zip(names, cols):
                np.save(f"{tag}_{name}.npy", arr)
        except OSError:  # /dev/shm too small: every rank draws the trace itself
            ok[0] = False
    dist.broadcast_object_list(ok, src=0)
    if not ok[0]:
        if rank == 0:
            for name in names:
                if os.path.exists(f"{tag}_{name}.npy"):
                    os.unlink(f"{tag}_{name}.npy")
        else:
            cols = generate_columns(ZipfSpec(schema(), ZIPF, n_batches * batch, seed))
    else:
        if rank != 0:
            cols = tuple(np.load(f"{tag}_{name}.npy", mmap_mode="r") for name in names)
        dist.barrier()  # every rank mapped the files: they can go (the mappings stay)
        if rank == 0:
            for name in names:
                os.unlink(f"{tag}_{name}.npy")
    rows, labels, dense = cols
    return batchify_columns(rows, labels, dense, batch)


def bench_config(world: int) -> dict:
    """The workload of one bench line, identical in both arms (ours and
    --impl reference) for the same N."""
    sc_rows = sum(CK_ROWS)
    return {"workload": WORKLOAD, "global_batch": BATCH * world, "per_gpu_batch": BATCH, "tables": len(CK_ROWS),
            "rows": sc_rows, "emb_dim": DIM, "cache_capacity_per_gpu": sc_rows // 100, "lookahead": "auto",
            "parallelism": "single" if world == 1 else f"{sharding(world)}-sharded x{world} (weak: {BATCH} examples/GPU)",
            "num_trainers": world,
            "l2": "flushed at the start of every timed iteration (256 MiB write inside the timed span)",
            "timing": "one CUDA-event span over K steps, end event after joining the plan and host-link streams",
            "mode": "stub-gradient (bit-exact)"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region by an
    in-process NVML thread (every ~2 ms).  NVML is initialised before the
    timed region starts, so no nvidia-smi process start-up (which takes the
    driver's locks for tens of milliseconds) lands inside it."""

    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20), ("hw_thermal_slowdown", 0x40),
               ("sw_power_cap", 0x4))
    PERIOD = float(os.environ.get("BAGPIPE_B200_CLOCK_PERIOD", "0.002"))  # seconds between NVML samples

    def __init__(self, index: int):
        self.index = index
        self.samples, self.reasons = [], set()
        self.smax = None
        self._stop = threading.Event()
        self._thr = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 -- no NVML: reported as unavailable
            self.nvml = None

    def _sample(self):
        nv = self.nvml
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM))
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
            for name, bit in self.REASONS:
                if bits & bit:
                    self.reasons.add(name)
        except Exception:  # noqa: BLE001
            pass

    def _loop(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(self.PERIOD)

    def start(self):
        if self.nvml is None:
            return
        self._thr = threading.Thread(target=self._loop, daemon=True)
        self._thr.start()

    def stop(self) -> dict:
        if self.nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["NVML unavailable"]}
        self._stop.set()
        if self._thr is not None:
            self._thr.join()
        if not self.samples:
            self._sample()
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.smax, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "NVML, sampled every ~2 ms during the timed region"}


# ------------------------------------------------------------- our engine
# Algorithmic bytes of the fused backward+SGD kernel per launch:
# per occurrence: position (4 B) + label (1 B); per unique key: CSR offset
# (4 B) + slot (4 B) + row read (4*D B) + row write (4*D B).
def stub_step_bytes(n_occ: int, u: int) -> int:
    return n_occ * 5 + u * (8 + 8 * DIM)


def count_launches(pipe, pos: int) -> int:
    """Kernels of our library launched by one engine step (torch profiler / CUPTI)."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        pipe.step(pos)
        torch.cuda.synchronize()
    n = 0
    for ev in prof.events():
        name = ev.name or ""
        if ev.device_type == torch.autograd.DeviceType.CUDA and ("bp::" in name or name.startswith("k_")):
            n += 1
    return n


# Kernels of the batch prep and of the Oracle Cacher planner (roofline_planner)
PREP_KERNELS = ("k_col_cluster_prep", "k_first_order", "k_occ_k_from_s", "k_prep_", "k_radix", "k_scan_onepass",
                "k_set_rank_bounds")
PLANNER_KERNELS = ("k_refill", "k_pop_fused")


def kernel_times(pipe, first: int, k: int) -> dict:
    """Device time per step of every kernel of our library over k engine
    steps (CUPTI through the torch profiler): {kernel name: us per step}."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(k):
            pipe.step(first + i, early=i < k - 1)
        torch.cuda.synchronize()
    out = {}
    for ev in prof.events():
        name = ev.name or ""
        if ev.device_type == torch.autograd.DeviceType.CUDA and ("bp::" in name or name.startswith("k_")):
            key = name.split("(")[0].replace("void ", "").replace("bp::", "")
            out[key] = out.get(key, 0.0) + ev.device_time / k
    return out


def prep_bytes(n_occ: int, u: int) -> int:
    """Algorithmic bytes of one batch prep: keys + labels
    read (9 B/occurrence), sorted positions + label bytes written (5 B), per
    unique key the sorted key, id, first-order key, both permutations and the
    CSR offset (32 B)."""
    return n_occ * 14 + u * 32


def planner_bytes(u: int, p: int, e: int) -> int:
    """Algorithmic bytes of refill + pop (SURVEY 8d planner row): tracker and
    flag updates of the batch entering the window (13 B/unique), the pop's
    tracker/flag reads + TTL and flag writes (21 B/unique), prefetch key/id/ttl
    (20 B each) and evict key/id (12 B each)."""
    return u * 34 + p * 20 + e * 12


def trace_ingest(batches) -> dict:
    """EMTRC1 file -> decoded device columns: the bench's
    batches written as a trace file, then streamed into pinned buffers, DMA'd
    and decoded on the GPU (ingest.read_trace_device); bytes/s of the file."""
    import tempfile

    from paper_2202_12429_b200.ingest import read_trace_device
    from paper_2202_12429_b200.traces import write_trace_columns

    rows = np.concatenate([b.rows for b in batches])
    labels = np.concatenate([b.labels for b in batches])
    dense = np.concatenate([b.dense for b in batches])
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "ck.trace")
        write_trace_columns(path, schema(), rows, labels, dense)
        read_trace_device(path)  # warm: allocations, page cache
        tr = read_trace_device(path)
    st = dict(tr.stats)
    st["note"] = (f"{len(batches)} CK batches ({st['records']} records x 261 B) from the page cache: readinto pinned "
                  "chunks, H2D DMA, bp_trace_decode (packed keys, occurrence labels, labels, dense)")
    return st


def _timed_steps(pipe, first: int, steps: int, flush_buf, torch, exclusive: int | None = None):
    """K steps as ONE span on the engine's compute stream, bracketed by
    device syncs: CUDA events, the end event recorded after the compute
    stream joined the engine's plan and host-link streams, so every kernel
    and copy the K steps issued is inside.  L2 is flushed at the start of
    every iteration by the engine itself (bp_engine_set_l2_flush: a 256 MiB
    memset on the compute stream; exclusive=1 also fences the plan and
    host-link streams around it), inside the span.  Returns (span ms, wall ms)."""
    from paper_2202_12429_b200 import _lib as L

    stream = pipe.stream
    if exclusive is None:
        exclusive = FLUSH_EXCLUSIVE
    L.check(pipe.lib.bp_engine_set_l2_flush(pipe.eng, L.ptr(flush_buf), flush_buf.numel(), exclusive),
            "bp_engine_set_l2_flush")
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    # no cyclic-GC pass (a multi-millisecond host stall) inside the short span
    gc.collect()
    gc.disable()
    try:
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        wait0 = pipe.host_wait_s
        start.record(stream)
        host_ts = []
        for i in range(steps):
            # the last timed step must not enqueue step K+1 ahead of time
            pipe.step(first + i, early=i < steps - 1)
            host_ts.append(time.perf_counter())
        L.check(pipe.lib.bp_engine_join(pipe.eng, L.stream_ptr(stream)), "bp_engine_join")
        end.record(stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - wall0) * 1e3
        pipe.timed_host_wait_ms = (pipe.host_wait_s - wait0) * 1e3
    finally:
        gc.enable()
    dump = os.environ.get("BAGPIPE_B200_BENCH_DUMP")  # debug: host time of every timed step
    if dump:
        with open(f"{dump}.steps.{os.environ.get('RANK', '0')}.{first}.json", "w") as fh:
            json.dump([round((t - wall0) * 1e3, 3) for t in host_ts], fh)
    L.check(pipe.lib.bp_engine_set_l2_flush(pipe.eng, None, 0, 0), "bp_engine_set_l2_flush")
    return start.elapsed_time(end), wall


def _stage_breakdown(pipe, first: int, k: int):
    """Per-stage device time over k extra (untimed) steps with the engine's
    stage events on; the timed region runs with them off (they cost host
    calls).  Returns ({stage: (ms per step, launches per step)}, k)."""
    pipe.lib.bp_engine_set_timing(pipe.eng, 1)
    pipe.stage_times()
    for i in range(k):
        pipe.step(first + i, early=i < k - 1)
    st = pipe.stage_times()
    pipe.lib.bp_engine_set_timing(pipe.eng, 0)
    return {name: (ms / k, n / k) for name, (ms, n) in st.items()}


def _flush_ms(flush_buf, steps: int, torch) -> float:
    """Device time of the per-iteration L2 flush alone (reported, not
    subtracted): the same memset, warmed up, timed over K repetitions."""
    for _ in range(3):
        flush_buf.zero_()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(steps):
        flush_buf.zero_()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e)


def run_ours(args, rank: int, world: int, local_rank: int) -> dict | None:
    import torch
    import torch.distributed as dist

    from paper_2202_12429_b200 import _lib as L
    from paper_2202_12429_b200.engine import EngineConfig, _Pipeline
    from paper_2202_12429_b200.shard import shard_batches, table_costs, table_shards

    if world > 1:
        # the host-link green partition (on by default) measured 4 % slower
        # at N=4 (tables per rank: the generic chunked prep keeps the SMs
        # busier) and equal at N=2, +5 % at N=1: the N>1 lines run without
        os.environ.setdefault("BAGPIPE_B200_GREEN_SMS", "0")
    L.lib()
    sc = schema()
    cap = sc.total_rows // 100
    steps, warm = args.steps, args.warmup
    link_probe = not args.no_link_probe
    n_batches = warm + (3 if link_probe else 2) * steps + 16
    # N>1 (weak scaling, the DLRM convention of a fixed per-GPU batch): the
    # global batch is N x 16,384 examples, its 26 tables dealt over the ranks;
    # every rank runs the whole pipeline for its tables of every example --
    # N x 16,384 x 26/N = the same 425,984 occurrences per step as one GPU --
    # with no data-path collective, and the same per-GPU HBM cache budget.
    gbatch = BATCH * world
    full = make_batches_shared(n_batches, args.seed, gbatch, rank, world)
    # tables dealt by their cost (occurrences + unique keys of the first
    # batch), largest first to the least-loaded rank
    shards = table_shards(sc.num_tables, world, table_costs(full[0])) if world > 1 else [list(range(sc.num_tables))]
    tables = shards[rank]
    if world == 1:
        batches = full
    elif sharding(world) == "row":
        from paper_2202_12429_b200.shard import row_shard_batches

        batches = row_shard_batches(full, world, rank)
    else:
        batches = shard_batches(full, tables)
    # DLRM mode (hybrid parallel) keeps whole tables per rank: its pooled-row
    # exchange is by table
    dlrm_batches = batches if (world == 1 or sharding(world) != "row") else shard_batches(full, tables)
    # N GPUs = the reference's N data-parallel trainers (rank r = examples
    # [r*B/N, (r+1)*B/N) of the global batch; gradients combined in rank order)
    trainers = int(os.environ.get("BAGPIPE_B200_BENCH_TRAINERS", str(world)))
    cfg = EngineConfig(cache_capacity=cap, batch_size=gbatch, lookahead=0, num_trainers=trainers, num_shards=1,
                       seed=11)

    # ---- value: inputs resident in HBM before timing
    dev_inputs = {}
    for i, b in enumerate(batches):
        keys, labels, _ = b.packed_occurrences()
        dev_inputs[i] = (torch.from_numpy(keys).cuda(), torch.from_numpy(labels).cuda())
    torch.cuda.synchronize()
    pipe = _Pipeline(cfg, sc, batches, None, None, device_inputs=dev_inputs, timing=True)
    lookahead0 = pipe.L0  # auto lookahead of this rank's trace
    pipe.begin()
    for pos in range(warm):
        pipe.step(pos)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    clocks = ClockSampler(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    pipe.lib.bp_engine_set_timing(pipe.eng, 0)
    clocks.start()
    ms, wall_ms = _timed_steps(pipe, warm, steps, flush_buf, torch)
    host_wait_ms = pipe.timed_host_wait_ms
    flush_ms = _flush_ms(flush_buf, steps, torch)
    clk = clocks.stop()
    records = pipe.records[warm:warm + steps]
    launches_per_step = count_launches(pipe, warm + steps)
    stages = _stage_breakdown(pipe, warm + steps + 1, 8)
    dump = os.environ.get("BAGPIPE_B200_BENCH_DUMP")  # debug: per-rank stage times
    if dump:
        with open(f"{dump}.rank{rank}.json", "w") as fh:
            json.dump({"rank": rank, "tables": list(tables), "ms_per_step": ms / steps,
                       "stages": {k: v[0] for k, v in stages.items()}}, fh)
    # the same K steps with every engine stream drained around each flush
    # (no overlap across iterations): reported beside the value
    ms_excl, _ = _timed_steps(pipe, warm + steps + 9, steps, flush_buf, torch, exclusive=1)
    nxt = warm + 2 * steps + 9
    ktimes = kernel_times(pipe, nxt, 4)
    nxt += 4
    # host link: the same steps with the store's fetch and write-back kernels
    # turned into no-ops (results become wrong; timing only).  The difference
    # is the part of the host link NOT hidden behind the compute stream.
    ms_nolink = None
    if link_probe:
        L.check(pipe.lib.bp_debug_skip_link(3), "bp_debug_skip_link")
        try:
            ms_nolink, _ = _timed_steps(pipe, nxt, steps, flush_buf, torch)
        finally:
            L.check(pipe.lib.bp_debug_skip_link(0), "bp_debug_skip_link")
    u_mean = statistics.mean(r.critical_size + r.background_size for r in records)
    pf_mean = statistics.mean(r.prefetch_count for r in records)
    ev_mean = statistics.mean(r.evicted_count for r in records)
    n_occ = int(statistics.mean(b.packed_occurrences()[0].size for b in batches[warm:warm + steps]))
    link_rows = np.zeros(2, dtype=np.int64)  # lazy prefetch over the run: host-link reads, GPU-computed inits
    pipe.lib.bp_store_link_counters(pipe.store.handle, link_rows.ctypes.data)
    host_frac = float(link_rows[0]) / max(int(link_rows.sum()), 1)
    green = np.zeros(2, dtype=np.int32)  # the host-link SM partition the driver made
    pipe.lib.bp_green_info(green.ctypes.data)
    pipe.close()
    del pipe

    # ---- e2e: host batches through the public engine API: every step's keys
    # and labels DMA'd from pinned host memory inside the timed span
    e2e_ms = 0.0
    e2e_h2d = 0
    if not args.no_e2e:
        for b in batches:
            b.pin_memory()
        # bytes DMA'd per step: the compact columnar upload (row ids at 1, 2
        # or 4 bytes per column + one label per example) where the batch has
        # one, else packed u64 keys + a label per occurrence
        def _h2d(b):
            pp = b._memo.get("pinned_planes")
            return pp[0].numel() + pp[1].numel() if pp is not None else b.packed_occurrences()[0].size * 9

        e2e_h2d = int(statistics.mean(_h2d(b) for b in batches[warm:warm + steps]))
        pipe2 = _Pipeline(cfg, sc, batches, None, None)
        pipe2.begin()
        for pos in range(warm):
            pipe2.step(pos)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e2e_ms, _ = _timed_steps(pipe2, warm, steps, flush_buf, torch)
        pipe2.close()
        del pipe2

    # ---- DLRM mode (N=1): the same engine feeding PyTorch MLPs (bf16 autocast)
    dlrm = None
    if not args.no_dlrm:
        dlrm = run_dlrm_mode(args, sc, dlrm_batches, cfg, flush_buf, torch, rank, world, len(tables), shards)

    ingest = None
    if world == 1 and not args.no_e2e:
        ingest = trace_ingest(full[:20])

    t = torch.tensor([ms, e2e_ms], device="cuda", dtype=torch.float64)
    by_rank = [ms / steps]
    if world > 1:
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        by_rank = [float(x[0]) / steps for x in allt]
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, e2e_max = float(t[0]), float(t[1])
    if rank != 0:
        return None
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    pl_prep_us = sum(v for k, v in ktimes.items() if k.startswith(PREP_KERNELS))
    pl_plan_us = sum(v for k, v in ktimes.items() if k.startswith(PLANNER_KERNELS))
    pl_bytes = prep_bytes(n_occ, int(u_mean)) + planner_bytes(int(u_mean), int(pf_mean), int(ev_mean))
    pl_ms = (pl_prep_us + pl_plan_us) * 1e-3
    roofline_planner = {
        "kernel": "batch prep (bp::k_col_cluster_prep + k_first_order) + Oracle Cacher (bp::k_refill + k_pop_fused)",
        "bound": "hbm (latency-bound: sort, scans, dependent random reads of the per-key planner state)",
        "bytes_per_step": pl_bytes, "ms_per_step": pl_ms, "unit": "GB/s",
        "achieved": pl_bytes / (pl_ms * 1e-3) / 1e9 if pl_ms else 0.0, "peak": None,
        "kernels_us_per_step": {k: round(v, 2) for k, v in ktimes.items()
                                if k.startswith(PREP_KERNELS + PLANNER_KERNELS)},
        "prep_us": pl_prep_us, "planner_us": pl_plan_us, "traffic": _planner_traffic(),
        "stage_span_ms": {"prep": stages["prep"][0], "planner": stages["planner"][0]},
        "timing": "CUPTI device time of the kernels over 4 engine steps; stage_span_ms = the engine's event "
                  "spans around the enqueue (include host enqueue gaps)",
        "note": "bytes: prep 14 B/occurrence + 32 B/unique, planner 34 B/unique + 20 B/prefetch + 12 B/evict "
                "(DESIGN.md section 3)"}
    roofline_planner.update(peak=hbm_peak, frac=roofline_planner["achieved"] / hbm_peak, peak_source=peak_src)
    stub_total, stub_launches = stages["trainer"]
    stub_ms = stub_total / max(stub_launches, 1e-9)
    stub_bytes = stub_step_bytes(n_occ, int(u_mean))
    stub_achieved = stub_bytes / (stub_ms * 1e-3) / 1e9 if stub_ms else 0.0
    fetch_total, fetch_n = stages["fetch"]  # per step
    samples = gbatch * steps  # one global batch per step across all ranks
    out = {
        "metric": METRIC,
        "value": samples / (ms_max * 1e-3),
        "value_kind": "stub-gradient engine samples/s (the reference's own run_pipeline arithmetic, bit-exact; "
                      "the like-for-like comparison with the CPU reference, SURVEY 8d) -- DLRM-mode samples/s "
                      "with MLPs is under 'dlrm'",
        "unit": "samples/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": warm,
        "ms_per_step": ms_max / steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (reference Zipf generator stream, columnar)",
        "config": bench_config(world),
        "lookahead_resolved": lookahead0,
        "e2e": None if args.no_e2e else {"value": samples / (e2e_max * 1e-3), "unit": "samples/s",
                                         "h2d_bytes_per_step": e2e_h2d, "d2h_bytes_per_step": 12 * 8 + 32},
        "roofline_stub_trainer": {"kernel": "bp::k_stub_step(+_long): fused gather + backward + rank-ordered combine"
                                            " + SGD", "bound": "hbm (latency-bound: per-key sequential f32 chains)",
                                  "achieved": stub_achieved, "peak": hbm_peak, "unit": "GB/s",
                                  "frac": stub_achieved / hbm_peak, "bytes_per_launch": stub_bytes,
                                  "ms_per_launch": stub_ms, "peak_source": peak_src},
        "stages_ms_per_step": {k: v[0] for k, v in stages.items()},
        "roofline_planner": roofline_planner,
        "host_link": {"prefetch_rows_per_step": pf_mean,
                      "prefetch_host_read_frac": host_frac,
                      "prefetch_link_gbs": pf_mean * host_frac * 64 / (fetch_total * 1e-3) / 1e9
                      if fetch_total else None,
                      "prefetch_peak_gbs": 19.5, "prefetch_peak_note": "zero-copy random 64 B rows",
                      "writeback_rows_per_step": ev_mean,
                      "writeback_link_gbs": ev_mean * DIM * 4 / (stages["flush"][0] * 1e-3) / 1e9
                      if stages["flush"][0] else None,
                      "writeback_peak_gbs": 56.5, "writeback_peak_note": "pinned memcpy D2H (copy-engine log append)",
                      "ms_per_step_link_disabled": None if ms_nolink is None else ms_nolink / steps,
                      "link_ms_per_step": stages["fetch"][0] + stages["flush"][0],
                      "hidden": None if ms_nolink is None else
                      max(0.0, min(1.0, 1.0 - max(0.0, ms - ms_nolink) / steps /
                                   max(stages["fetch"][0] + stages["flush"][0], 1e-9))),
                      "hidden_note": "1 - (ms/step with the host link - ms/step with the store's fetch and "
                                     "write-back kernels disabled) / (fetch + write-back stage ms/step)",
                      "prefetch_note": "rows never written back are computed on the GPU (functional init, "
                                       "store.py:106-129); only written rows are read over the host link",
                      "peak_note": "pinned memcpy 55.5 GB/s H2D, 56.5 D2H; zero-copy random 64 B rows 18.7-25 GB/s "
                                   "(tools/hostlink_peak.py)",
                      "green_partition_sms": {"link": int(green[0]), "rest": int(green[1])}},
        "trace_ingest": ingest,
        "gpu_launches": launches_per_step * steps,
        "clocks": clk,
        "wall_ms_timed_region": wall_ms,
        # host time blocked waiting for step results inside the span: near 0
        # means the host loop, not the device, paces the steps
        "host_wait_ms_timed_region": round(host_wait_ms, 3),
        "l2_flush_ms_per_step": flush_ms / steps,
        "ms_per_step_exclusive_flush": ms_excl / steps,
        "ms_per_step_by_rank": by_rank,
    }
    if dlrm is not None:
        out["dlrm"] = dlrm["summary"]
        out["roofline"] = dlrm["roofline"]
        out["roofline"]["peak"] = hbm_peak
        out["roofline"]["frac"] = out["roofline"]["achieved"] / hbm_peak
        out["roofline"]["peak_source"] = peak_src
        for part in (dlrm.get("roofline_parts") or {}).values():
            part.update(peak=hbm_peak, frac=part["achieved"] / hbm_peak, peak_source=peak_src,
                        frac_cupti=part["achieved_cupti"] / hbm_peak if part.get("achieved_cupti") else None)
        out["roofline_parts"] = dlrm.get("roofline_parts")
        if dlrm.get("event_span_null_kernel_us"):
            out["event_span_null_kernel_us"] = dlrm["event_span_null_kernel_us"]
    else:
        out["roofline"] = dict(out["roofline_stub_trainer"], bound="hbm")
    return out


def run_dlrm_mode(args, sc, batches, cfg, flush_buf, torch, rank=0, world=1, local_tables=26, shards=None) -> dict:
    """DLRM mode; N > 1 = hybrid parallel (hybrid.py): this rank's table shard
    through the engine over the global batch, all-to-all of pooled rows and
    their gradients, data-parallel MLPs with a mean all-reduce."""
    import torch.distributed as dist

    from paper_2202_12429_b200.dlrm import DLRMConfig, DLRMTrainer
    from paper_2202_12429_b200.engine import _Pipeline
    from paper_2202_12429_b200.hybrid import EmbeddingExchange

    steps, warm = args.steps, args.warmup
    dcfg = DLRMConfig(emb_optimizer="sgd", emb_lr=0.01, mlp_lr=0.01, mlp_dtype="bf16",
                      sorted_grad=os.environ.get("BAGPIPE_B200_SORTED_GRAD", "1") != "0")
    ex = None
    if world > 1:
        from paper_2202_12429_b200.hybrid import PeerExchange

        # NVLink peer-memory exchange fused into the EmbeddingBag kernels
        # (default) or the NCCL all-to-all version
        if os.environ.get("BAGPIPE_B200_EXCHANGE", "peer") == "peer":
            ex = PeerExchange(sc.num_tables, DIM, rank, world, BATCH, shards=shards)
        else:
            ex = EmbeddingExchange(sc.num_tables, DIM, rank, world, shards=shards)
    trainer = DLRMTrainer(dcfg, sc.num_dense, sc.num_tables, DIM, exchange=ex)
    dev_inputs = {}
    for i, b in enumerate(batches):
        keys, labels, _ = b.packed_occurrences()
        dev_inputs[i] = (torch.from_numpy(keys).cuda(), torch.from_numpy(labels).cuda())
        trainer.set_device_dense(i, torch.from_numpy(np.ascontiguousarray(b.dense, dtype=np.float32)).cuda(),
                                 torch.from_numpy(b.labels.astype(np.float32)).cuda())
    pipe = _Pipeline(cfg, sc, batches, None, None, device_inputs=dev_inputs, timing=True, trainer=trainer)
    pipe.begin()
    for pos in range(warm):
        pipe.step(pos)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    pipe.lib.bp_engine_set_timing(pipe.eng, 0)
    ms, _ = _timed_steps(pipe, warm, steps, flush_buf, torch)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    records = pipe.records[warm:warm + steps]
    stages = _stage_breakdown(pipe, warm + steps, 8)
    # CUPTI device time of the same kernels inside 4 more steps (no event
    # brackets: the kernel alone, still beside the step's other streams)
    ktimes = kernel_times(pipe, warm + steps + 8, 4)
    ev_over = event_overhead_us(pipe.stream, torch) if world == 1 else None
    u_mean = statistics.mean(r.critical_size + r.background_size for r in records)
    n_occ = BATCH * world * local_tables
    # "trainer" spans: the EmbeddingBag forward, "trainer_bwd": its backward
    # + optimizer (one each per step); per step
    fwd_span, bwd_span = stages["trainer"], stages["trainer_bwd"]
    spans = (fwd_span[0] + bwd_span[0], fwd_span[1] + bwd_span[1])
    # forward N_occ*(64 row read + 64 pooled write + 4 index)
    fwd_bytes = n_occ * (8 * DIM + 4)
    losses = trainer.loss_history()
    pipe.close()
    del pipe
    return {"summary": {"value": BATCH * world * steps / (ms * 1e-3), "unit": "samples/s", "ms_per_step": ms / steps,
                        "parallelism": "single" if world == 1 else
                        f"hybrid: table-sharded embeddings + data-parallel MLP x{world}, "
                        f"{'NVLink peer-memory' if hasattr(ex, 'rows_x') else 'NCCL all-to-all'} exchange",
                        "mlp": "PyTorch, bf16 compute copy + fp32 master SGD, one CUDA graph per step (13-512-256-64-16 / 367-1024-1024-512-256-1)",
                        "embedding_optimizer": "sgd", "final_loss": losses[-1] if losses else None,
                        "embedding_stage_ms_per_step": spans[0]},
            "roofline": {"kernel": "bp::k_embbag_fwd_rows_v4 + k_bwd_reduce_reg + k_bwd_apply (EmbeddingBag fwd + sorted-gradient "
                                   "bwd+SGD on cached rows)",
                         "bound": "hbm", "bytes_per_step": fwd_bytes + bwd_bytes(n_occ, int(u_mean)),
                         "ms_per_step": spans[0], "launches_per_step": 2, "unit": "GB/s",
                         "achieved": (fwd_bytes + bwd_bytes(n_occ, int(u_mean))) / (spans[0] * 1e-3) / 1e9
                         if spans[0] else 0.0,
                         "traffic": _traffic(),
                         "note": "SURVEY 8(d) algorithmic bytes: forward N_occ*(64 row read + 64 pooled write + 4 "
                                 "index) + backward N_occ*(64 gradient read + 4 index) + U*(64 read + 64 write)"},
            # the two halves of the pair above, each timed by its own stage
            # events in the same steps
            # (N > 1: the peer-exchange variants, their spans include the
            # device-side barriers of the exchange)
            # span of a trivial kernel between two events on the same stream
            # (idle / busy): the part of each span above that is not kernel time
            "event_span_null_kernel_us": ev_over,
            "roofline_parts": None if world > 1 else {
                "gather": _part("bp::k_embbag_fwd_rows_v4 (EmbeddingBag forward: gather + pooling)",
                                fwd_bytes, fwd_span, "k_embbag_fwd_rows_v4", ktimes),
                "scatter": _part(SCATTER_LABEL, bwd_bytes(n_occ, int(u_mean)), bwd_span,
                                 ("k_embbag_bwd_staged", "k_bwd_reduce_reg", "k_bwd_apply"), ktimes,
                                 traffic_names=("k_bwd_reduce_reg", "k_bwd_apply"))}}


# the sorted-gradient backward kernels of the default variant (CUPTI times
# of every listed kernel are summed)
SCATTER_LABEL = ("bp::k_embbag_bwd_staged (sorted-gradient segmented scatter-add + SGD in place); "
                 "variants 8/9: bp::k_bwd_reduce_reg + bp::k_bwd_apply")


def event_overhead_us(stream, torch) -> dict:
    """CUDA-event span of a trivial kernel on `stream`: begin event, one
    tiny kernel, end event, back to back from the host -- with the stream
    idle (as at a host-paced stage start) and busy behind a 256 MiB memset
    (the stream ahead of the host).  What a stage span adds to a kernel's
    own duration (tools/mb/event_overhead.py)."""
    import statistics

    x = torch.zeros(1, device="cuda")
    big = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {}
    for mode in ("idle", "busy"):
        spans = []
        for _ in range(30):
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                if mode == "busy":
                    big.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                x.add_(1.0)
                b.record(stream)
            b.synchronize()
            spans.append(a.elapsed_time(b) * 1e3)
        out[mode] = round(statistics.median(spans), 2)
    del big
    return out


def _part(kernel: str, nbytes: int, span, ncu_name, ktimes: dict | None = None, traffic_names=None) -> dict:
    """One half of the EmbeddingBag pair: achieved = algorithmic bytes / the
    launch's CUDA-event span on the compute stream (the spec's measure; the
    span includes the launch gap behind the begin event), plus the CUPTI
    kernel duration inside the step for comparison."""
    ms = span[0]
    traffic = None
    for rnd in ("round2", "round1"):
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", rnd, "traffic.json")))["dram_bytes_per_launch"]
            # the default launch shape's kernels (all of them, summed)
            names = traffic_names or ncu_name
            traffic = sum(v for k, v in tr.items() if k.startswith(names)) or None
        except (OSError, KeyError, ValueError):
            continue
        if traffic is not None:
            break
    kus = None
    if ktimes:
        kus = sum(v for k, v in ktimes.items() if k.startswith(ncu_name)) or None
    return {"kernel": kernel, "bound": "hbm", "bytes_per_launch": nbytes, "ms_per_launch": ms,
            "launches_per_step": span[1], "unit": "GB/s", "achieved": nbytes / (ms * 1e-3) / 1e9 if ms else 0.0,
            "traffic": traffic, "kernel_us_cupti_in_step": kus,
            "achieved_cupti": nbytes / (kus * 1e-6) / 1e9 if kus else None}


def _traffic():
    """DRAM bytes (read + write) per step of the EmbeddingBag kernels from the
    committed ncu --set full capture (profiles/round2/traffic.json)."""
    for rnd in ("round2", "round1"):
        try:
            return json.load(open(os.path.join(ROOT, "profiles", rnd, "traffic.json")))[
                "embbag_fwd_bwd_dram_bytes_per_step"]
        except (OSError, KeyError, ValueError):
            continue
    return None


def _planner_traffic():
    """DRAM bytes per step of the prep + planner kernels (ncu --set full of
    tools/planner_bench.py, profiles/round2/traffic.json)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "round2", "traffic.json")))[
            "prep_planner_dram_bytes_per_step"]
    except (OSError, KeyError, ValueError):
        return None


def bwd_bytes(n_occ: int, u: int) -> int:
    return n_occ * (4 * DIM + 4) + u * (8 * DIM)


# ------------------------------------------------------- CPU oracle timing
def cpu_oracle(steps: int, warmup: int, seed: int) -> dict:
    """Time the CPU port of the reference pipeline (oracle/) on CK batches."""
    from oracle import bagpipe_oracle as O

    sc = schema()
    batches = make_batches(warmup + steps + 10, seed)
    cap = sc.total_rows // 100
    run = O.OraclePipeline(batches, CK_ROWS, DIM, 11, 1, cap, 7 if SHAPE == "ck" else 0, 0.25)
    run.begin()
    for pos in range(warmup):
        run.step(pos)
    t0 = time.perf_counter()
    for pos in range(warmup, warmup + steps):
        run.step(pos)
    dt = time.perf_counter() - t0
    return {"value": BATCH * steps / dt, "unit": "samples/s", "cores": 1, "kind": "port",
            "sample": f"{steps} CK iterations (after {warmup} warm-up) of the oracle pipeline port, "
                      f"numpy single-threaded, {dt:.1f} s", "ms_per_step": dt * 1e3 / steps}


def main():
    args = parse()
    apply_shape(args.shape)
    if args.shape != "ck":
        args.no_dlrm = True  # the DLRM-mode line is the Criteo-Kaggle model
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        if rank != 0:
            return 0
        cb = cpu_oracle(args.steps, max(args.warmup, 1), args.seed)
        line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "samples/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms_per_step"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (reference Zipf generator stream, columnar)",
                "config": bench_config(world if world > 1 else args.gpus),
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": cb["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0
    import torch

    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = run_ours(args, rank, world, local_rank)
    if out is not None:
        if not args.no_cpu_baseline and world == 1:
            cb = cpu_oracle(args.cpu_steps, 2, args.seed)
            out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        elif not args.no_cpu_baseline:
            out["cpu_baseline"] = None
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
