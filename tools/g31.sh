timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_matrix.py tests/test_gpu_engine.py -x > gpurun_out/g31_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g31_pytest.log
for c in C5 C4 C3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g31_bench_$c.json 2> gpurun_out/g31_bench_$c.err
done
