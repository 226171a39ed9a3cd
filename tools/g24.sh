for c in C5 C4; do EDX_GREEDY_STATS=1 EDX_GRAPH=0 timeout 600 python tools/one_iteration.py --config $c > gpurun_out/g24_stats_$c.log 2>&1; done
