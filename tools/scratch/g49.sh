timeout 1800 python -m pytest -q -p no:cacheprovider -m gpu tests > gpurun_out/g49_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g49_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g49_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/g49_bench.json 2> gpurun_out/g49_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/g49_bench_ref.json 2> gpurun_out/g49_bench_ref.err
