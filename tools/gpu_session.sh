#!/bin/bash
# One gpurun session: GPU tests + bench lines, outputs under gpurun_out/$TAG*.
# usage: tools/gpu_session.sh TAG "pytest-args" "bench-configs"
TAG=${1:-s}
PYARGS=${2:-"tests -m gpu"}
CONFIGS=${3:-"C3"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
if [ "$PYARGS" != "none" ]; then
  timeout 1800 python -m pytest $PYARGS -q --durations=20 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
  tail -3 gpurun_out/${TAG}_pytest.log
fi
for c in $CONFIGS; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 $BENCH_EXTRA > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo "bench $c rc=$?"
done
