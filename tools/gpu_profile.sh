#!/bin/bash
# Round profiling on the GPU box (run from the repo root under gpurun):
# plain runs first, then the ncu launch lists and the --set full captures.
#   bash tools/gpu_profile.sh [out_dir]
set -u
OUT=${1:-gpurun_out/prof}
mkdir -p "$OUT"
timeout 300 python tools/profile_step.py --steps 3 --nvtx --engine-flush 0 > "$OUT/plain_stub.log" 2>&1 || exit 11
timeout 300 python tools/profile_step.py --steps 3 --nvtx --engine-flush 0 --dlrm > "$OUT/plain_dlrm.log" 2>&1 || exit 12
timeout 300 python tools/planner_bench.py --nvtx --no-prof --batches 16 > "$OUT/plain_planner.log" 2>&1 || exit 13
# launch lists (serialised, cold cache: shares, not absolute times)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed_step/" \
  --csv --log-file "$OUT/launches_stub.csv" python tools/profile_step.py --steps 3 --nvtx --engine-flush 0 \
  > "$OUT/ncu_l1.log" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed_step/" \
  --csv --log-file "$OUT/launches_dlrm.csv" python tools/profile_step.py --steps 3 --nvtx --engine-flush 0 --dlrm \
  > "$OUT/ncu_l2.log" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "planner_batch/" \
  --csv --log-file "$OUT/launches_planner.csv" python tools/planner_bench.py --nvtx --no-prof --batches 16 \
  > "$OUT/ncu_l3.log" 2>&1
# full captures of the roofline kernels and the prep / planner kernels
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed_step/" \
  -k regex:"k_embbag|k_interact|k_bwd_reduce_reg|k_bwd_apply" -c 8 -f -o "$OUT/full_dlrm" python tools/profile_step.py --steps 1 --nvtx \
  --engine-flush 0 --dlrm > "$OUT/ncu_f1.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "planner_batch/" \
  -k regex:"k_col_cluster|k_first_order|k_pop_fused|k_refill" -c 4 -f -o "$OUT/full_planner" \
  python tools/planner_bench.py --nvtx --no-prof --batches 13 > "$OUT/ncu_f2.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed_step/" \
  -k regex:"k_stub_step|k_store_fetch|k_evict_planned|k_insert|k_apply" -c 10 -f -o "$OUT/full_stub" \
  python tools/profile_step.py --steps 2 --nvtx --engine-flush 0 > "$OUT/ncu_f3.log" 2>&1
echo done
