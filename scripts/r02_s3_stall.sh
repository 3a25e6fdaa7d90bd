#!/bin/bash
# virtual-rank forward progress with pool-drawn dW / write-back streams: the 2-rank tests that stalled,
# 8 times each, then the whole GPU suite twice
O=gpurun_out/r02s3stall; mkdir -p $O
for i in 1 2 3 4 5 6 7 8; do
  timeout 600 python -m pytest tests/test_gpu_nvls.py tests/test_gpu_accum.py tests/test_gpu_model.py -q -p no:cacheprovider \
      -k "gated_off or duplicated or matches_oracle" > $O/loop_$i.log 2>&1
  echo "loop $i rc=$? $(grep -E 'passed|failed' $O/loop_$i.log | tail -1)" >> $O/summary.txt
done
for rep in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_$rep.log 2>&1
  echo "gpu suite $rep rc=$? $(grep -E 'passed|failed' $O/pytest_gpu_$rep.log | tail -1)" >> $O/summary.txt
done
