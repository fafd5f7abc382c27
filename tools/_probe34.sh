set -u
mkdir -p gpurun_out/p34
timeout 300 python tools/kernel_bench.py > gpurun_out/p34/kb.json 2> gpurun_out/p34/kb.err; echo "kb rc=$?"
for rep in 1 2; do
timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-link-probe > gpurun_out/p34/b_$rep.json 2> gpurun_out/p34/b_$rep.err; echo "b rc=$?"
done
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/p34/tests.log 2>&1; echo "tests rc=$?"
