EDX_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "edx.iter/" -k regex:k_big_select -c 1 -o gpurun_out/g48_bigsel python tools/one_iteration.py --config C5 --batch 65536 --workers 8 --prefill 18 > gpurun_out/g48_ncu.log 2>&1
echo "rc=$?"
