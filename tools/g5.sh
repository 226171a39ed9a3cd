tools/gpu_session.sh g5 "tests -m gpu" "C3"
BENCH_EXTRA="--spread-ids --no-ncu" tools/gpu_session.sh g5spread none "C3"
python tools/solver_profile.py --config C3 --prefill 3 --reps 2 > gpurun_out/g5_solver.jsonl 2>&1
timeout 1200 python tools/solver_table2.py --parity-max 2048 > gpurun_out/g5_table2.jsonl 2> gpurun_out/g5_table2.err
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/g5_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/g5_memcheck.log
echo done
