timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_engine.py tests/test_gpu_scale.py -x -k "c5 or engine" > gpurun_out/g42_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g42_pytest.log
for c in C5 C4 C3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g42_bench_$c.json 2> gpurun_out/g42_bench_$c.err
done
EDX_HEAD_OVERLAP=0 timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g42_benchh_C5.json 2> gpurun_out/g42_benchh_C5.err
