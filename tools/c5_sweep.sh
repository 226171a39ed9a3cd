#!/bin/bash
# The C5 sweep grid (BASELINE.json configs[4]: batch 4K-64K x workers 8-64,
# greedy, 800K-entry caches) on the GPUs of this box: one bench line per point,
# N = 1 and (when present) every larger power of two as torchrun ranks.
# usage (via gpurun): tools/c5_sweep.sh TAG
TAG=${1:-c5s}
G=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
for R in 4096 16384 65536; do
  for n in 8 16 32 64; do
    for N in 1 2 4 8; do
      [ $N -gt $G ] && continue
      out=gpurun_out/${TAG}_b${R}_w${n}_g${N}.json
      if [ $N -eq 1 ]; then
        timeout 600 python bench.py --config C5 --batch $R --workers $n --steps 10 --warmup 3 \
          --no-cpu-baseline --no-ncu > $out 2> $out.err
      else
        timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
          --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N --config C5 \
          --batch $R --workers $n --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > $out 2> $out.err
      fi
      echo "R=$R n=$n N=$N rc=$?"
    done
  done
done
