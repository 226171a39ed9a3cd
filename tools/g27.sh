timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_matrix.py tests/test_gpu_engine.py tests/test_gpu_golden.py -x > gpurun_out/g27_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g27_pytest.log
for c in C5 C4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g27_bench_$c.json 2> gpurun_out/g27_bench_$c.err
done
EDX_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "edx.iter/" --csv --log-file gpurun_out/g27_launches_C5.csv python tools/one_iteration.py --config C5 > gpurun_out/g27_l_C5.log 2>&1
