#!/bin/bash
# Multi-GPU bench lines (run via gpurun --gpus 4): N = 2 and 4 for C2 (the driver's
# scaling config), C4 and C5, launched like the driver (torchrun, one rank per GPU).
set -u
mkdir -p gpurun_out
for N in 2 4; do
  for c in C2 C4 C5; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29600 + N)) bench.py --gpus $N --config $c > gpurun_out/sc_${c}_n$N.json \
      2> gpurun_out/sc_${c}_n$N.err
    echo "$c n=$N rc=$?"
  done
done
