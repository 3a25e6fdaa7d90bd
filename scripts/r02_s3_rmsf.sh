#!/bin/bash
# register-resident RMSNorm forward (group of G warps per row): GPU suite, ncu of one launch, A/B
O=gpurun_out/r02s3rmsf; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "gpu suite rc=$? $(grep -E 'passed|failed' $O/pytest_gpu.log | tail -1)" > $O/summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rmsnorm_fwd_group -s 4 -c 1 \
    -o $O/rms_fwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_full.out 2>&1
echo "ncu full rc=$?" >> $O/summary.txt
for rep in 1 2; do
  DC_RMSNORM_TWO_PASS=1 timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/prev_$rep.json 2> $O/prev_$rep.err
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/new_$rep.json 2> $O/new_$rep.err
done
echo "ab done" >> $O/summary.txt
