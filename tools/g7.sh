for c in C2 C3 C4; do python tools/solver_profile.py --config $c --prefill 3 --reps 2 >> gpurun_out/g7_solver.jsonl 2>> gpurun_out/g7_solver.err; done
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_matrix.py tests/test_gpu_solver_layouts.py tests/test_gpu_engine.py "tests/test_gpu_scale.py::test_c2_alpha_one" "tests/test_gpu_scale.py::test_c3_evicting_steady_state" > gpurun_out/g7_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g7_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/g7_bench_C3.json 2> gpurun_out/g7_bench_C3.err
