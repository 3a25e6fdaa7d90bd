#!/bin/bash
# Adam sqrt(v)/c by the reciprocal + 2 FMA residuals (abtree/, -DDC_ADAM_RCP_DIV) vs div.rn (this tree), in-step A/B
O=gpurun_out/r02s3rcp; mkdir -p $O
(cd abtree && timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "rs_adam" > ../$O/pytest_rcp.log 2>&1)
echo "rcp rs_adam tests rc=$? $(tail -1 $O/pytest_rcp.log)" > $O/summary.txt
for rep in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/div_$rep.json 2> $O/div_$rep.err
  (cd abtree && timeout 600 python bench.py --no-cpu-baseline --steps 10) > $O/rcp_$rep.json 2> $O/rcp_$rep.err
done
