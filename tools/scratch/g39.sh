timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_matrix.py tests/test_gpu_engine.py tests/test_gpu_golden.py -x > gpurun_out/g39_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g39_pytest.log
for c in C3 C2; do python tools/solver_profile.py --config $c --prefill 3 --reps 2 >> gpurun_out/g39_solver.jsonl 2>> gpurun_out/g39_solver.err; done
for c in C5 C4 C3 C2 C1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g39_bench_$c.json 2> gpurun_out/g39_bench_$c.err
done
for c in C5 C3 C1; do
  EDX_HEAD_OVERLAP=0 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g39_benchh_$c.json 2> gpurun_out/g39_benchh_$c.err
done
