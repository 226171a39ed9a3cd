EDX_GRAPH=0 timeout 600 python tools/one_iteration.py --config C5 > gpurun_out/g16_plain.log 2>&1 && \
EDX_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "edx.iter/" -k regex:'k_greedy$' -c 1 \
  -o gpurun_out/g16_greedy_C5 python tools/one_iteration.py --config C5 > gpurun_out/g16_ncu.log 2>&1
echo "rc=$?"
EDX_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "edx.iter/" -k regex:'k_cost_build' -c 1 \
  -o gpurun_out/g16_k1_C5 python tools/one_iteration.py --config C5 > gpurun_out/g16_ncu_k1.log 2>&1
echo "rc=$?"
