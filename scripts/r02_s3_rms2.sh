#!/bin/bash
# one-pass RMSNorm backward v2 (dh, x, dres issued together; dg partials in shared memory)
O=gpurun_out/r02s3rms2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > $O/pytest_sub.log 2>&1
echo "subset rc=$? $(grep -E 'passed|failed' $O/pytest_sub.log | tail -1)" > $O/summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rmsnorm_bwd_fused -s 4 -c 1 \
    -o $O/rms_fused python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_full.out 2>&1
echo "ncu full rc=$?" >> $O/summary.txt
for rep in 1 2; do
  DC_RMSNORM_TWO_PASS=1 timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/two_$rep.json 2> $O/two_$rep.err
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/one_$rep.json 2> $O/one_$rep.err
done
echo "ab done" >> $O/summary.txt
