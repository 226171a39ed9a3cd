EDX_SOLVER_TIMING=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hungarian_blocks_mw -s 3 -c 1 \
  -o gpurun_out/g28_k6_c3 python tools/solver_profile.py --config C3 --prefill 3 --reps 1 > gpurun_out/g28_ncu_k6.log 2>&1
echo "k6 rc=$?"
