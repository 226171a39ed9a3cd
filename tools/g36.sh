timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests -x > gpurun_out/g36_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g36_pytest.log
for c in C4 C3; do python tools/solver_profile.py --config $c --prefill 3 --reps 2 >> gpurun_out/g36_solver.jsonl 2>> gpurun_out/g36_solver.err; done
for c in C4 C5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g36_bench_$c.json 2> gpurun_out/g36_bench_$c.err
done
