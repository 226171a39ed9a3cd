for c in C3 C4 C5; do timeout 600 python tools/k1_stats.py --config $c >> gpurun_out/g13_k1stats.jsonl 2>> gpurun_out/g13_k1stats.err; done
for c in C5 C4; do
EDX_GRAPH=0 timeout 600 python tools/one_iteration.py --config $c > gpurun_out/g13_plain_$c.log 2>&1 && \
EDX_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "edx.iter/" -k regex:k_cost_build -c 1 \
  -o gpurun_out/g13_k1_$c python tools/one_iteration.py --config $c > gpurun_out/g13_ncu_k1_$c.log 2>&1
echo "$c rc=$?"
done
