python tools/scratch/hung_timing.py > gpurun_out/g37_hung_default.log 2>&1
CUDA_MODULE_LOADING=EAGER python tools/scratch/hung_timing.py > gpurun_out/g37_hung_eager.log 2>&1
(cd tests/cpp && timeout 900 ./reftests/acceptance > ../../gpurun_out/g37_acc_default.log 2>&1)
(cd tests/cpp && CUDA_MODULE_LOADING=EAGER timeout 900 ./reftests/acceptance > ../../gpurun_out/g37_acc_eager.log 2>&1)
