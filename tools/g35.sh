for c in C5 C3; do
timeout 900 ncu --graph-profiling graph --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g35_graph_$c.csv python tools/one_iteration.py --config $c > gpurun_out/g35_g_$c.log 2>&1
done
EDX_SOLVER_TIMING=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hungarian_blocks_mw -s 3 -c 1 \
  -o gpurun_out/g35_k6_c3 python tools/solver_profile.py --config C3 --prefill 3 --reps 1 > gpurun_out/g35_ncu_k6.log 2>&1
