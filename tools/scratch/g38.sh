timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_matrix.py tests/test_gpu_engine.py tests/test_gpu_golden.py tests/test_gpu_solver_layouts.py -x > gpurun_out/g38_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g38_pytest.log
for c in C3 C2; do python tools/solver_profile.py --config $c --prefill 3 --reps 2 >> gpurun_out/g38_solver.jsonl 2>> gpurun_out/g38_solver.err; done
for c in C5 C4 C3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g38_bench_$c.json 2> gpurun_out/g38_bench_$c.err
done
EDX_HEAD_OVERLAP=0 timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g38_benchh_C5.json 2> gpurun_out/g38_benchh_C5.err
EDX_PDL=0 timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g38_benchp_C5.json 2> gpurun_out/g38_benchp_C5.err
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests/test_reference_suite.py tests/test_gpu_scale.py > gpurun_out/g38_pytest2.log 2>&1; echo "rc=$?" >> gpurun_out/g38_pytest2.log
