#!/bin/bash
# N>1 bench code paths on ONE GPU (gloo, every rank on cuda:0): correctness of the plumbing only --
# the numbers are meaningless (ranks share the GPU).
set -e
for n in 2 4 8; do
  PBSA_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --steps 3 --warmup 3 --no-cpu \
    2>&1 | grep -E '^\{|Error|error' | head -5
done
PBSA_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29599 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --scaling weak \
  2>&1 | grep -E '^\{|Error|error' | head -5
