timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_engine.py tests/test_gpu_matrix.py tests/test_gpu_golden.py tests/test_gpu_scale.py tests/test_gpu_solver_layouts.py -x > gpurun_out/g34_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g34_pytest.log
for c in C3 C4 C2; do python tools/solver_profile.py --config $c --prefill 3 --reps 2 >> gpurun_out/g34_solver.jsonl 2>> gpurun_out/g34_solver.err; done
for c in C5 C4 C3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g34_bench_$c.json 2> gpurun_out/g34_bench_$c.err
done
for c in C5 C3; do
EDX_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "edx.iter/" --csv --log-file gpurun_out/g34_launches_$c.csv python tools/one_iteration.py --config $c > gpurun_out/g34_l_$c.log 2>&1
done
