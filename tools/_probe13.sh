set -u
mkdir -p gpurun_out/p13
timeout 300 python tools/profile_step.py --steps 4 --dlrm --engine-flush 0 --trace gpurun_out/p13/dlrm_trace.json > gpurun_out/p13/prof.log 2>&1; echo "prof rc=$?"
