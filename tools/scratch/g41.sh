timeout 1800 python -m pytest -q -p no:cacheprovider -m gpu tests > gpurun_out/g41_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g41_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g41_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/g41_bench.json 2> gpurun_out/g41_bench.err
for c in C5 C1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g41_bench_$c.json 2> gpurun_out/g41_bench_$c.err; done
