tools/gpu_session.sh g4 "tests -m gpu" "C5 C1"
for c in C2 C3 C4; do python tools/solver_profile.py --config $c --prefill 3 --reps 2 >> gpurun_out/g4_solver.jsonl 2>> gpurun_out/g4_solver.err; done
for c in C3 C4; do EDX_MW_BPW=2 python tools/solver_profile.py --config $c --prefill 3 --reps 2 >> gpurun_out/g4_solver.jsonl 2>> gpurun_out/g4_solver.err; done
timeout 900 python tools/solver_table2.py --parity-max 2048 > gpurun_out/g4_table2.jsonl 2> gpurun_out/g4_table2.err
echo done
