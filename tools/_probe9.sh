set -u
mkdir -p gpurun_out/p9
timeout 600 python -m pytest tests/test_gpu_dlrm.py tests/test_gpu_ck_dlrm.py -x -q > gpurun_out/p9/dlrm.log 2>&1; echo "dlrm rc=$?"
timeout 300 python tools/kernel_bench.py > gpurun_out/p9/kernel.json 2> gpurun_out/p9/kernel.err; echo "kernel rc=$?"
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/p9/bench.json 2> gpurun_out/p9/bench.err; echo "bench rc=$?"
