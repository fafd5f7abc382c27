"""Per-stream kernel timeline of a chrome trace written by profile_step.py --trace.

  python tools/timeline.py trace.json [first_ms] [span_ms]
"""

from __future__ import annotations

import json
import sys


def main():
    path = sys.argv[1]
    ev = json.load(open(path))
    ev = ev["traceEvents"] if isinstance(ev, dict) else ev
    ks = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "ts" in e]
    ks.sort(key=lambda e: e["ts"])
    t0 = ks[0]["ts"]
    first = float(sys.argv[2]) * 1e3 if len(sys.argv) > 2 else 0.0
    span = float(sys.argv[3]) * 1e3 if len(sys.argv) > 3 else 3e3
    for e in ks:
        ts = e["ts"] - t0
        if ts < first or ts > first + span:
            continue
        name = e["name"].split("(")[0].replace("void ", "")[:48]
        stream = e.get("args", {}).get("stream", e.get("tid"))
        print(f"{ts:10.1f} {e.get('dur', 0):8.1f}  s{stream:<4} {name}")


if __name__ == "__main__":
    main()
