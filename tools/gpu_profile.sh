#!/bin/bash
# Round profiling on the GPU box (run from the repo root under gpurun):
# plain runs first, then the ncu launch list and the --set full captures.
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
timeout 300 python tools/profile_step.py --steps 3 --nvtx > "$OUT/plain_stub.log" 2>&1 || exit 11
timeout 300 python tools/profile_step.py --steps 3 --nvtx --dlrm > "$OUT/plain_dlrm.log" 2>&1 || exit 12
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed_step/" \
  --csv --log-file "$OUT/launches_stub.csv" python tools/profile_step.py --steps 3 --nvtx > "$OUT/ncu_l1.log" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed_step/" \
  --csv --log-file "$OUT/launches_dlrm.csv" python tools/profile_step.py --steps 3 --nvtx --dlrm > "$OUT/ncu_l2.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed_step/" \
  -k regex:"k_stub_step|k_prep_table_sort|k_store_fetch|k_store_write|k_log_commit|k_evict_planned|k_insert|k_pop|k_apply" \
  -c 16 -f -o "$OUT/full_stub" python tools/profile_step.py --steps 2 --nvtx > "$OUT/ncu_f1.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed_step/" \
  -k regex:"k_embbag|k_interact" -c 6 -f -o "$OUT/full_dlrm" python tools/profile_step.py --steps 1 --nvtx --dlrm \
  > "$OUT/ncu_f2.log" 2>&1
echo done
