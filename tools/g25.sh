for c in C5 C4 C3; do
EDX_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "edx.iter/" --csv --log-file gpurun_out/g25_launches_$c.csv python tools/one_iteration.py --config $c > gpurun_out/g25_l_$c.log 2>&1
done
