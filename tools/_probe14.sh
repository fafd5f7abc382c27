set -u
mkdir -p gpurun_out/p14
rm -f gpurun_out/p14/out.jsonl
timeout 300 python -m pytest tests/test_gpu_dlrm.py -x -q -k "sorted_gradient" > gpurun_out/p14/dlrm.log 2>&1; echo "dlrm rc=$?"
run() { env "$@" timeout 300 python tools/embbag_instep.py --steps 30 >> gpurun_out/p14/out.jsonl 2>> gpurun_out/p14/err.log; }
run BAGPIPE_B200_BWD_VARIANT=6
run BAGPIPE_B200_BWD_VARIANT=4
run BAGPIPE_B200_BWD_VARIANT=0
timeout 300 python tools/kernel_bench.py > gpurun_out/p14/kernel.json 2> gpurun_out/p14/kernel.err; echo "kernel rc=$?"
echo done
