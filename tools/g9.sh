for c in C3 C4 C2; do python tools/solver_profile.py --config $c --prefill 3 --reps 2 >> gpurun_out/g9_solver.jsonl 2>> gpurun_out/g9_solver.err; done
EDX_MW_BPW=2 python tools/solver_profile.py --config C3 --prefill 3 --reps 2 >> gpurun_out/g9_solver.jsonl 2>> gpurun_out/g9_solver.err
for c in C5 C3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g9_bench_$c.json 2> gpurun_out/g9_bench_$c.err
done
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_matrix.py tests/test_gpu_scale.py tests/test_gpu_solver_layouts.py > gpurun_out/g9_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g9_pytest.log
