#!/bin/bash
# Multi-GPU CUDA-graph A/B (run via gpurun --gpus 4): the sharded-engine parity
# test at 2 and 4 ranks with the graph path, then bench lines at N = 2, 4 for
# C2 and C5 with EDX_MULTI_GRAPH=1 (graph) and 0 (eager).
set -u
mkdir -p gpurun_out
for W in 2 4; do
  EDX_TEST_WORLD=$W timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/mg_test_w$W.log 2>&1
  echo "parity w=$W rc=$?"
done
for N in 2 4; do
  for c in C2 C5; do
    for G in 1 0; do
      EDX_MULTI_GRAPH=$G timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
        --master-addr 127.0.0.1 --master-port $((29700 + N)) bench.py --gpus $N --config $c \
        --no-cpu-baseline > gpurun_out/mg_${c}_n${N}_g$G.json 2> gpurun_out/mg_${c}_n${N}_g$G.err
      echo "$c n=$N graph=$G rc=$?"
    done
  done
done
