timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests -x > gpurun_out/g33_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g33_pytest.log
for c in C5 C4; do EDX_GREEDY_STATS=1 EDX_GRAPH=0 timeout 600 python tools/one_iteration.py --config $c > gpurun_out/g33_stats_$c.log 2>&1; done
for c in C5 C4 C3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g33_bench_$c.json 2> gpurun_out/g33_bench_$c.err
  EDX_GAP_SORT=merge timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g33_benchm_$c.json 2> gpurun_out/g33_benchm_$c.err
done
EDX_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "edx.iter/" --csv --log-file gpurun_out/g33_launches_C5.csv python tools/one_iteration.py --config C5 > gpurun_out/g33_l_C5.log 2>&1
