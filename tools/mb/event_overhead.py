"""CUDA-event span of (almost) nothing: record, tiny kernel, record on one
stream, back to back from the host, while the stream is idle and while it
is busy behind a long kernel.  The idle case shows what an event-timed
stage span adds to a kernel's own duration (launch latency behind the
begin event); the busy case shows the span of the same launch once the
stream runs ahead of the host.

  python tools/mb/event_overhead.py
"""

import json
import statistics

import torch


def main():
    s = torch.cuda.Stream()
    x = torch.zeros(1, device="cuda")
    big = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {}
    for mode in ("idle", "busy"):
        spans = []
        for _ in range(50):
            torch.cuda.synchronize()
            with torch.cuda.stream(s):
                if mode == "busy":
                    big.zero_()  # ~40 us of work ahead of the events
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                x.add_(1.0)
                b.record(s)
            b.synchronize()
            spans.append(a.elapsed_time(b) * 1e3)
        out[mode + "_us_median"] = round(statistics.median(spans), 2)
        out[mode + "_us_min"] = round(min(spans), 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
