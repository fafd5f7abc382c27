"""SMs the driver gives a green-context partition for each requested count
(`BAGPIPE_B200_GREEN_SMS`): one engine per request, each in its own
interpreter (the partition is process-wide), reported by bp_green_info.

  python tools/mb/green_granularity.py > profiles/round2/green_granularity.json
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import test_gpu_green as T  # noqa: E402


def main():
    out = {}
    for req in (1, 2, 4, 6, 8, 12, 16, 24):
        r = T._run(16, str(req))
        out[str(req)] = {"link_sms": r["hot"], "rest_sms": r["rest"]}
        print(req, out[str(req)], file=sys.stderr, flush=True)
    print(json.dumps({"requested_to_made": out, "note": "D=16 engine, bp_green_info after run_pipeline"}))


if __name__ == "__main__":
    main()
