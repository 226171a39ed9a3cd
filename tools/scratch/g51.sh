python tools/solver_profile.py --config C3 --prefill 3 --reps 2 >> gpurun_out/g51_solver.jsonl 2>> gpurun_out/g51_solver.err
EDX_MW_BPW=2 python tools/solver_profile.py --config C3 --prefill 3 --reps 2 >> gpurun_out/g51_solver.jsonl 2>> gpurun_out/g51_solver.err
