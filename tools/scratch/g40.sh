timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_matrix.py tests/test_gpu_engine.py tests/test_gpu_golden.py -x > gpurun_out/g40_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g40_pytest.log
for c in C1 C2 C3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g40_bench_$c.json 2> gpurun_out/g40_bench_$c.err
done
