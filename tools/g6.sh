set -u
mkdir -p gpurun_out
for c in C2 C3 C4; do python tools/solver_profile.py --config $c --prefill 3 --reps 2 >> gpurun_out/g6_solver.jsonl 2>> gpurun_out/g6_solver.err; done
timeout 1200 python -m pytest tests/test_gpu_solver_layouts.py -q -p no:cacheprovider > gpurun_out/g6_layouts.log 2>&1; echo "layouts rc=$?" >> gpurun_out/g6_layouts.log
for c in C3 C4 C1 C2; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g6_bench_$c.json 2> gpurun_out/g6_bench_$c.err
  EDX_K1=lane timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g6_lane_$c.json 2> gpurun_out/g6_lane_$c.err
done
for c in C5 C4 C3; do
  EDX_GRAPH=0 timeout 900 ncu --nvtx --nvtx-include "edx.iter/" --metrics gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/g6_launches_$c.csv \
    python tools/one_iteration.py --config $c > gpurun_out/g6_ncu_$c.log 2>&1
  echo "launches $c rc=$?"
done
echo done
