#!/bin/bash
# Collects the round's measured evidence on one B200 into gpurun_out/ (run via gpurun):
# the GPU parity suite, smoke, bench lines for every workload (C3 = the default), the
# reference arm on the default workload, the launch list of one steady-state iteration
# per workload, and full ncu captures of the cost build (K1), the exact solver (K6) and
# the greedy (K4).  Each ncu pass runs only after the same command has exited 0 without
# ncu (the bench lines above).
set -u
mkdir -p gpurun_out
T=${TAG:-ev}
timeout 1800 python -m pytest -q -p no:cacheprovider -m gpu tests > gpurun_out/${T}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke rc=$?"
for c in C3 C1 C2 C4 C5; do
  timeout 900 python bench.py --config $c > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
  echo "bench $c rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_ref_C3.json 2> gpurun_out/${T}_bench_ref.err
echo "reference rc=$?"
for c in C3 C5 C4 C2; do
  EDX_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx \
    --nvtx-include "edx.iter/" --csv --log-file gpurun_out/${T}_launches_$c.csv \
    python tools/one_iteration.py --config $c > gpurun_out/${T}_l_$c.log 2>&1
  echo "launches $c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${T}_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --no-ncu > gpurun_out/${T}_ncu_launch.log 2>&1
echo "bench launch list rc=$?"
for c in C3 C4 C5; do
  EDX_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on --nvtx \
    --nvtx-include "edx.iter/" -k regex:k_cost_build -c 1 -o gpurun_out/${T}_k1_$c \
    python tools/one_iteration.py --config $c > gpurun_out/${T}_ncu_k1_$c.log 2>&1
  echo "k1 $c rc=$?"
done
EDX_SOLVER_TIMING=0 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_hungarian_blocks_mw -s 3 -c 1 -o gpurun_out/${T}_k6_c3 \
  python tools/solver_profile.py --config C3 --prefill 3 --reps 1 > gpurun_out/${T}_ncu_k6.log 2>&1
echo "k6 rc=$?"
EDX_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on --nvtx \
  --nvtx-include "edx.iter/" -k regex:'k_greedy$' -c 1 -o gpurun_out/${T}_k4_c5 \
  python tools/one_iteration.py --config C5 > gpurun_out/${T}_ncu_k4.log 2>&1
echo "k4 rc=$?"
for c in C2 C3 C4; do
  python tools/solver_profile.py --config $c --prefill 3 --reps 2 >> gpurun_out/${T}_solver.jsonl 2>> gpurun_out/${T}_solver.err
done
