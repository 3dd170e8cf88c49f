#!/bin/bash
# Functional check of every sharded bench path with 2 ranks on ONE GPU (gloo, CSRK_BENCH_ONE_GPU=1):
# the numbers are not bench values (two ranks share one GPU; gloo stages through the host).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
port=29611
for w in cfg2 cfg3 cfg4 cfg5; do
  port=$((port + 1))
  CSRK_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port $port bench.py --gpus 2 --workload $w --steps 2 --warmup 3 \
    --no-cpu-baseline --no-e2e > gpurun_out/dist_smoke_$w.json 2> gpurun_out/dist_smoke_$w.err
  echo "$w rc=$? $(tail -c 250 gpurun_out/dist_smoke_$w.json)"
done
