timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_multi.py > gpurun_out/g32_multi.log 2>&1; echo "rc=$?" >> gpurun_out/g32_multi.log
bash tools/scale.sh g32 "C3 C5 C4" > gpurun_out/g32_scale.log 2>&1
