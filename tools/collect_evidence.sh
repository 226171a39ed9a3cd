#!/bin/bash
# Collects the round's measured evidence on one B200 into gpurun_out/ (run via gpurun):
# bench lines for every workload, the reference arm, the kernel launch list of the
# default bench command, and full ncu captures of the cost build (K1) for its traffic
# and of the exact solver (K6).  Each ncu pass runs only after the same command has
# exited 0 without ncu (the bench lines above).
set -u
mkdir -p gpurun_out
for c in C2 C1 C3 C4 C5; do
  timeout 600 python bench.py --config $c > gpurun_out/ev_bench_$c.json 2> gpurun_out/ev_bench_$c.err
  echo "bench $c rc=$?"
done
timeout 600 python bench.py --impl reference > gpurun_out/ev_bench_ref_C2.json 2> gpurun_out/ev_bench_ref.err
echo "reference rc=$?"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dadd_peak tools/dadd_peak.cu && \
  ./tools/dadd_peak > gpurun_out/ev_dadd_peak.json 2>&1; echo "dadd rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/ev_launches_c2.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ev_ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cost_build_warp -s 22 -c 2 \
  -o gpurun_out/ev_k1_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_k1c2.log 2>&1
echo "k1 c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cost_build_wide -s 4 -c 1 \
  -o gpurun_out/ev_k1_c4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_k1c4.log 2>&1
echo "k1 c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cost_build_wide64 -s 3 -c 1 \
  -o gpurun_out/ev_k1_c5 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_k1c5.log 2>&1
echo "k1 c5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hungarian_blocks_mw -s 22 -c 1 \
  -o gpurun_out/ev_k6_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_k6c2.log 2>&1
echo "k6 c2 rc=$?"
