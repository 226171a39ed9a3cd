timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_matrix.py tests/test_gpu_engine.py tests/test_gpu_ids.py tests/test_gpu_dropin.py "tests/test_gpu_scale.py::test_c5_corner" > gpurun_out/g8_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g8_pytest.log
for c in C5 C1 C2 C4 C3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g8_bench_$c.json 2> gpurun_out/g8_bench_$c.err
done
EDX_GRAPH=0 timeout 900 ncu --nvtx --nvtx-include "edx.iter/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g8_launches_C5.csv python tools/one_iteration.py --config C5 > gpurun_out/g8_ncu_C5.log 2>&1
