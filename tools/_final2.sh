set -u
mkdir -p gpurun_out/f2
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/f2/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/f2/bench.json 2> gpurun_out/f2/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/f2/bench_ref.json 2> gpurun_out/f2/bench_ref.err; echo "ref rc=$?"
timeout 300 python tools/kernel_bench.py > gpurun_out/f2/kb.json 2> gpurun_out/f2/kb.err; echo "kb rc=$?"
timeout 900 python bench.py > gpurun_out/f2/bench2.json 2> gpurun_out/f2/bench2.err; echo "bench2 rc=$?"
