EDX_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "edx.iter/" -k regex:'k_greedy' -c 2 \
  -o gpurun_out/g19_greedy_C5 python tools/one_iteration.py --config C5 > gpurun_out/g19_ncu.log 2>&1
echo "rc=$?"
