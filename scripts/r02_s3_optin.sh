#!/bin/bash
# the opt-in virtual-rank stress cases (graph replay at N = 2 / 4, copy-engine gathers at N = 2 / 4), 4 runs each
O=gpurun_out/r02s3optin; mkdir -p $O
for i in 1 2 3 4; do
  DC_TEST_GRAPH_N=1 DC_TEST_CE=1 DC_SPIN_MS=5000 timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_model.py \
      -q -p no:cacheprovider -k "virtual_ranks_bitexact or copy_engine_gather" > $O/run_$i.log 2>&1
  echo "run $i rc=$? $(grep -E 'passed|failed' $O/run_$i.log | tail -1)" >> $O/summary.txt
  grep -E "^FAILED|^E  .*DC_" $O/run_$i.log | head -4 >> $O/summary.txt
done
