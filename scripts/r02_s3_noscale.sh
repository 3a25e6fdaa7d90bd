#!/bin/bash
# N = 1 bulk update without the 1/N multiply (this tree) vs with it (abtree/ = HEAD~): in-step A/B + rs_adam tests
O=gpurun_out/r02s3noscale; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -q -p no:cacheprovider -k "rs_adam or matches_oracle" > $O/pytest.log 2>&1
echo "tests rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
for rep in 1 2 3; do
  (cd abtree && timeout 600 python bench.py --no-cpu-baseline --steps 10) > $O/prev_$rep.json 2> $O/prev_$rep.err
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/new_$rep.json 2> $O/new_$rep.err
done
