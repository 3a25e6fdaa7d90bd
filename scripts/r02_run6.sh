#!/bin/bash
# bulk-copy (TMA-staged) push: parity, T_c sweep vs the 16-byte-store push at virtual N = 2 / 8, ncu of both;
# config-5 proxy (70B layers at N = 1 just past the device: small adaptive offload)
O=gpurun_out/r02run6; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -k "ag_" -q -p no:cacheprovider > $O/ag_tests.log 2>&1
echo "ag tests rc=$? $(tail -1 $O/ag_tests.log)" > $O/summary.txt
timeout 1500 python scripts/ag_sweep.py --worlds 2,8 --modes sm,bulk --max-log2 31 --steps 5 --out $O/ag_sweep_bulk.json > $O/ag_sweep.txt 2>&1
echo "sweep rc=$?" >> $O/summary.txt
for m in sm bulk; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:ag_push -c 4 -o $O/ag_push_n8_$m \
    python scripts/ag_sweep.py --ncu-push 8 --max-log2 30 --modes $m > $O/ncu_ag_$m.txt 2>&1
  echo "ncu $m rc=$?" >> $O/summary.txt
done
for L in 13 14; do
  timeout 900 python bench.py --offload --model llama3-70b --layers $L --batch 1 --steps 3 --warmup 3 --no-cpu-baseline \
      > $O/offload_70b_L$L.json 2> $O/offload_70b_L$L.err
  echo "offload L=$L rc=$?" >> $O/summary.txt
done
