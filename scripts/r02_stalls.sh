#!/bin/bash
# Forward-progress evidence: repeated runs of the N > 1
# configurations that stalled intermittently in round 1.
mkdir -p gpurun_out/stalls
R=gpurun_out/stalls/summary.txt
: > $R
bash scripts/share_loop.sh ${1:-10}
cp -r gpurun_out/sl gpurun_out/stalls/share_gpu
echo "share-gpu bench (2 processes on cuda:0):" >> $R
cat gpurun_out/sl/res.txt >> $R
for i in $(seq 1 ${2:-5}); do
  DC_TEST_GRAPH_N=1 DC_TEST_CE=1 timeout 600 python -m pytest tests/test_gpu_graph.py tests/test_gpu_model.py \
      -k "virtual_ranks or copy_engine" -q -p no:cacheprovider > gpurun_out/stalls/graph_ce_$i.log 2>&1
  echo "graph-N + copy-engine N=4 run $i rc=$? $(tail -1 gpurun_out/stalls/graph_ce_$i.log)" >> $R
done
