#!/bin/bash
# glue kernels with 32-bit index math: A/B against the previous commit (abtree2), alternating; GPU suite
O=gpurun_out/r02run19; mkdir -p $O
for rep in 1 2; do
  (cd abtree2 && timeout 600 python bench.py --no-cpu-baseline --steps 10) > $O/prev_$rep.json 2> $O/prev_$rep.err
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/new_$rep.json 2> $O/new_$rep.err
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "gpu suite rc=$? $(grep -E 'passed|failed' $O/pytest_gpu.log | tail -1)" > $O/summary.txt
