timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_matrix.py tests/test_gpu_engine.py tests/test_gpu_golden.py -x > gpurun_out/g23_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g23_pytest.log
for c in C5 C4; do EDX_GREEDY_STATS=1 EDX_GRAPH=0 timeout 600 python tools/one_iteration.py --config $c > gpurun_out/g23_stats_$c.log 2>&1; done
for c in C5 C4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g23_bench_$c.json 2> gpurun_out/g23_bench_$c.err
done
