# N-GPU bench lines (table- and row-sharded), the reference arm and the
# multi-GPU tests on one box:  gpurun --gpus N -- 'bash tools/multi_gpu.sh N'
set -u
N=$1
mkdir -p gpurun_out/m$N
for sh in table row; do
BAGPIPE_B200_SHARDING=$sh timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus $N > gpurun_out/m$N/bench_$sh.json 2> gpurun_out/m$N/bench_$sh.err; echo "bench $sh rc=$?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus $N --impl reference > gpurun_out/m$N/ref.json 2> gpurun_out/m$N/ref.err; echo "ref rc=$?"
timeout 900 python -m pytest tests -q -m gpu -k "hybrid or shard or peer or dist" > gpurun_out/m$N/tests.log 2>&1; echo "tests rc=$?"
