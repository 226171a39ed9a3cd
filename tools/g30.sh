timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_matrix.py tests/test_gpu_scale.py tests/test_gpu_solver_layouts.py -x > gpurun_out/g30_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g30_pytest.log
for c in C3 C4 C2; do python tools/solver_profile.py --config $c --prefill 3 --reps 2 >> gpurun_out/g30_solver.jsonl 2>> gpurun_out/g30_solver.err; done
