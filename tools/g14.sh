timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_matrix.py tests/test_gpu_engine.py -x > gpurun_out/g14_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g14_pytest.log
for c in C3 C4 C5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g14_bench_$c.json 2> gpurun_out/g14_bench_$c.err
  EDX_K1_WIDE=1 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g14_benchw_$c.json 2> gpurun_out/g14_benchw_$c.err
done
