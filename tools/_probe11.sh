set -u
mkdir -p gpurun_out/p11
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_reduce|k_bwd_apply|k_embbag_bwd_staged|k_embbag_fwd_rows" -c 4 -f -o gpurun_out/p11/bwd python tools/kernel_bench.py --reps 1 > gpurun_out/p11/ncu.log 2>&1; echo "ncu rc=$?"
