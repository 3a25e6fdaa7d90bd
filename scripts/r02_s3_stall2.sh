#!/bin/bash
# the NVLS-gated-off 2-rank test 16 times (every failing rank's wait record in the message)
O=gpurun_out/${OUT:-r02s3stall2}; mkdir -p $O
for i in $(seq 1 16); do
  timeout 300 python -m pytest tests/test_gpu_nvls.py -q -p no:cacheprovider -k "gated_off" > $O/loop_$i.log 2>&1
  echo "loop $i rc=$? $(grep -E 'passed|failed' $O/loop_$i.log | tail -1)" >> $O/summary.txt
  grep -E "^E  .*DC_" $O/loop_$i.log | head -2 >> $O/summary.txt
done
