#!/bin/bash
# GPU suite twice (virtual-rank steps now return after the device step: no two rank sets in flight)
O=gpurun_out/r02s3suite; mkdir -p $O
for rep in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_$rep.log 2>&1
  echo "gpu suite $rep rc=$? $(grep -E 'passed|failed' $O/pytest_gpu_$rep.log | tail -1)" >> $O/summary.txt
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$? $(tail -1 $O/smoke.log)" >> $O/summary.txt
