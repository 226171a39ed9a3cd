for n in 8; do
EDX_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "edx.iter/" --csv --log-file gpurun_out/g43_launches_w$n.csv python tools/one_iteration.py --config C5 --batch 65536 --workers $n --prefill 18 > gpurun_out/g43_l_$n.log 2>&1
done
