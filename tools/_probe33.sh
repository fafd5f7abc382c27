set -u
mkdir -p gpurun_out/p33
./tools/mb/atomic_probe > gpurun_out/p33/atomic.jsonl 2>&1; echo "atomic rc=$?"
timeout 300 python tools/kernel_bench.py > gpurun_out/p33/kb.json 2> gpurun_out/p33/kb.err; echo "kb rc=$?"
for rep in 1 2 3; do
timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-link-probe --no-dlrm > gpurun_out/p33/b_$rep.json 2> gpurun_out/p33/b_$rep.err; echo "b rc=$?"
done
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_units.py -x -q > gpurun_out/p33/tests.log 2>&1; echo "tests rc=$?"
