#!/bin/bash
# one-pass RMSNorm backward (register-resident rows) vs the two-pass form: alternating A/B on one box,
# GPU suite, ncu --set full of the new kernel and a launch list of the default command
O=gpurun_out/r02s3rms; mkdir -p $O
for rep in 1 2; do
  DC_RMSNORM_TWO_PASS=1 timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/two_$rep.json 2> $O/two_$rep.err
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/one_$rep.json 2> $O/one_$rep.err
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "gpu suite rc=$? $(grep -E 'passed|failed' $O/pytest_gpu.log | tail -1)" > $O/summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rmsnorm_bwd_fused -s 4 -c 2 \
    -o $O/rms_fused python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_full.out 2>&1
echo "ncu full rc=$?" >> $O/summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"rmsnorm|colsum" -c 40 --csv --log-file $O/rms_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_l.out 2>&1
DC_RMSNORM_TWO_PASS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"rmsnorm|colsum" -c 40 --csv --log-file $O/rms_launches_two.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_l2.out 2>&1
echo "ncu launches rc=$?" >> $O/summary.txt
