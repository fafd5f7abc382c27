"""Host-link (PCIe) peaks on the GPU box: pinned memcpy H2D/D2H and the
zero-copy row gather/scatter kernels of the store at 64 B rows.

  python tools/hostlink_peak.py   -> one JSON line
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2202_12429_b200.store import ShardedStore  # noqa: E402


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def main():
    out = {}
    nbytes = 256 << 20
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    out["memcpy_h2d_gbs"] = nbytes / timed(lambda: d.copy_(h, non_blocking=True)) / 1e9
    out["memcpy_d2h_gbs"] = nbytes / timed(lambda: h.copy_(d, non_blocking=True)) / 1e9
    sc = bench.schema()
    store = ShardedStore(sc, 1, 11)
    rng = np.random.default_rng(0)
    from paper_2202_12429_b200 import _lib as L

    for blocks in (8, 16, 32, 64, 148):
        L.check(L.lib().bp_set_link_config(blocks, 256, 0), "bp_set_link_config")
        ids = np.sort(rng.integers(0, sc.total_rows, 35_000)).astype(np.uint32)
        d_ids = torch.from_numpy(ids).cuda()
        rows = torch.empty((35_000, sc.emb_dim), dtype=torch.float32, device="cuda")
        out[f"gather_random_35000_blocks{blocks}_gbs"] = 35_000 * 64 / timed(
            lambda: store.fetch_ids_async(d_ids, 35_000)) / 1e9
        out[f"scatter_random_35000_blocks{blocks}_gbs"] = 35_000 * 64 / timed(
            lambda: store.write_ids_async(d_ids, rows, 35_000)) / 1e9
    L.check(L.lib().bp_set_link_config(32, 256, 0), "bp_set_link_config")
    # host worker pool gather/scatter of random rows of the pinned table (DMA link mode)
    import ctypes as C

    table = L.lib().bp_store_host_table(store.handle)
    if table:
        ids = np.sort(rng.integers(0, sc.total_rows, 35_000)).astype(np.uint32)
        for threads in (1, 2, 4, 8, 12):
            for op, name in ((0, "gather"), (1, "scatter")):
                sec = C.c_double()
                L.check(L.lib().bp_host_rows_bench(table, sc.emb_dim, ids.ctypes.data, 35_000, threads, op,
                                                   C.byref(sec)), "bp_host_rows_bench")
                out[f"host_{name}_35000_threads{threads}_us"] = sec.value * 1e6
    for n in (35_000, 1_000_000):
        for kind in ("random", "sequential"):
            ids = rng.integers(0, sc.total_rows, n) if kind == "random" else np.arange(n)
            ids = np.sort(ids).astype(np.uint32)
            d_ids = torch.from_numpy(ids).cuda()
            rows = torch.empty((n, sc.emb_dim), dtype=torch.float32, device="cuda")
            t = timed(lambda: store.fetch_ids_async(d_ids, n))
            out[f"zero_copy_gather_{kind}_{n}_gbs"] = n * 64 / t / 1e9
            t = timed(lambda: store.write_ids_async(d_ids, rows, n))
            out[f"zero_copy_scatter_{kind}_{n}_gbs"] = n * 64 / t / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
