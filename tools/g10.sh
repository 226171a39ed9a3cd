for c in C2 C3; do python tools/solver_profile.py --config $c --prefill 3 --reps 2 >> gpurun_out/g10_solver.jsonl 2>> gpurun_out/g10_solver.err; done
EDX_SOLVER_TIMING=0 python tools/solver_profile.py --config C3 --prefill 3 --reps 1 > gpurun_out/g10_plain.log 2>&1 && \
EDX_SOLVER_TIMING=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hungarian_blocks_mw -c 1 \
  -o gpurun_out/g10_k6_c3 python tools/solver_profile.py --config C3 --prefill 3 --reps 1 > gpurun_out/g10_ncu_k6.log 2>&1
echo "k6 rc=$?"
EDX_GRAPH=0 python tools/one_iteration.py --config C3 > gpurun_out/g10_plain2.log 2>&1 && \
EDX_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cost_build -s 4 -c 1 \
  -o gpurun_out/g10_k1_c3 python tools/one_iteration.py --config C3 > gpurun_out/g10_ncu_k1.log 2>&1
echo "k1 rc=$?"
