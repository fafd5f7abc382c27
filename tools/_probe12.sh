set -u
mkdir -p gpurun_out/p12
timeout 600 python -m pytest tests/test_gpu_dlrm.py -x -q > gpurun_out/p12/dlrm.log 2>&1; echo "dlrm rc=$?"
timeout 300 python tools/kernel_bench.py > gpurun_out/p12/kernel.json 2> gpurun_out/p12/kernel.err; echo "kernel rc=$?"
for v in 0 4; do for g in 0 3; do
BAGPIPE_B200_BWD_VARIANT=$v BAGPIPE_B200_LINK_GATE=$g timeout 600 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-link-probe > gpurun_out/p12/bench_v${v}_g${g}.json 2> gpurun_out/p12/bench_v${v}_g${g}.err; echo "bench $v $g rc=$?"
done; done
