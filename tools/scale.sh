#!/bin/bash
# Multi-GPU bench lines: N = 1, 2, 4, ... up to the GPUs of this
# box, for the given configs; one torchrun per N (rank per GPU over NCCL).
# usage (on a gpurun --gpus G box): tools/scale.sh TAG "C4 C5"
TAG=${1:-sc}
CONFIGS=${2:-"C4 C5"}
G=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
for c in $CONFIGS; do
  for N in 1 2 4 8; do
    [ $N -gt $G ] && continue
    if [ $N -eq 1 ]; then
      timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-ncu \
        > gpurun_out/${TAG}_${c}_n1.json 2> gpurun_out/${TAG}_${c}_n1.err
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
        --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --config $c \
        --steps 20 --warmup 5 --no-cpu-baseline --no-ncu \
        > gpurun_out/${TAG}_${c}_n$N.json 2> gpurun_out/${TAG}_${c}_n$N.err
    fi
    echo "$c N=$N rc=$?"
  done
done
