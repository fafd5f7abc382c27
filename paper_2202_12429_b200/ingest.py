"""EMTRC1 trace ingest into HBM (reference traces.py:231-296).

The reference decodes a trace record by record into Python ``Example``
objects (~1 s per Criteo-Kaggle batch).  Here the record bytes stream from
the file straight into pinned host buffers (``readinto``, two buffers in
flight), are DMA'd to HBM, and ``bp_trace_decode`` turns each chunk into the
engine's device batch layout -- packed keys in occurrence order, one label
byte per occurrence, labels and dense features -- so a run can start from a
file without materialising any per-example host object.
"""

from __future__ import annotations

import time

import torch

from . import _lib as L
from .errors import TraceFormatError
from .traces import Schema, _read_header


class DeviceTrace:
    """A decoded trace resident in HBM (occurrence-major columns)."""

    def __init__(self, schema: Schema, n: int, keys, occ_labels, labels, dense, stats: dict):
        self.schema, self.n = schema, n
        self.keys, self.occ_labels, self.labels, self.dense = keys, occ_labels, labels, dense
        self.stats = stats

    def batch_inputs(self, batch_size: int, first: int = 0) -> dict:
        """{position: (d_keys, d_occ_labels)} views of consecutive batches, the
        engine's device_inputs (zero-copy slices)."""
        t = self.schema.num_tables
        out = {}
        for pos, e0 in enumerate(range(0, self.n, batch_size)):
            e1 = min(self.n, e0 + batch_size)
            out[first + pos] = (self.keys[e0 * t:e1 * t], self.occ_labels[e0 * t:e1 * t])
        return out


def read_trace_device(path: str, chunk_bytes: int = 64 << 20, stream=None) -> DeviceTrace:
    """Stream an EMTRC1 file into HBM and decode it there.  ``stats`` holds
    the file bytes, the wall-clock ingest time (file -> decoded columns in
    HBM) and the device time of the decode kernels."""
    lib = L.lib()
    stream = stream or torch.cuda.current_stream()
    with open(path, "rb") as fh:
        schema, count = _read_header(fh)
        offset = fh.tell()
    t, d = schema.num_tables, schema.num_dense
    rb = 1 + 4 * d + 8 * t
    per = max(1, chunk_bytes // rb)
    dev = "cuda"
    keys = torch.empty(count * t, dtype=torch.uint64, device=dev)
    occ = torch.empty(count * t, dtype=torch.uint8, device=dev)
    labels = torch.empty(count, dtype=torch.uint8, device=dev)
    dense = torch.empty((count, d), dtype=torch.float32, device=dev)
    pinned = [torch.empty(per * rb, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    raw = [torch.empty(per * rb, dtype=torch.uint8, device=dev) for _ in range(2)]
    freed = [None, None]
    spans = []
    t0 = time.perf_counter()
    with open(path, "rb", buffering=0) as fh:
        fh.seek(offset)
        done, k = 0, 0
        while done < count:
            m = min(per, count - done)
            i = k & 1
            if freed[i] is not None:
                freed[i].synchronize()  # the DMA that last read this pinned buffer is done
            view = pinned[i].numpy()[: m * rb]
            got = fh.readinto(memoryview(view))
            if got != m * rb:
                raise TraceFormatError("truncated trace")
            with torch.cuda.stream(stream):
                raw[i][: m * rb].copy_(pinned[i][: m * rb], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
                freed[i] = ev
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                L.check(lib.bp_trace_decode(L.ptr(raw[i]), m, d, t, L.ptr(keys) + done * t * 8,
                                            L.ptr(occ) + done * t, L.ptr(labels) + done,
                                            (L.ptr(dense) + done * d * 4) if d else None,
                                            L.stream_ptr(stream)), "bp_trace_decode")
                b.record(stream)
                spans.append((a, b))
            done += m
            k += 1
    stream.synchronize()
    wall = time.perf_counter() - t0
    dec_ms = sum(a.elapsed_time(b) for a, b in spans)
    nbytes = count * rb
    stats = {"records": count, "bytes": nbytes, "wall_s": wall, "ingest_gbs": nbytes / wall / 1e9 if wall else None,
             "decode_ms": dec_ms, "decode_gbs": nbytes / (dec_ms * 1e-3) / 1e9 if dec_ms else None,
             "chunks": k}
    return DeviceTrace(schema, count, keys, occ, labels, dense, stats)


__all__ = ["DeviceTrace", "read_trace_device"]
