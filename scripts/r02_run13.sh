#!/bin/bash
# the N-rank bench launch path end to end on one GPU (processes time-slicing cuda:0): N = 4 and 8
O=gpurun_out/r02run13; mkdir -p $O
for n in 4 8; do
  CUDA_DEVICE_MAX_CONNECTIONS=8 timeout 900 python bench.py --gpus $n --share-gpu --layers 2 --batch 1 --steps 2 \
      --warmup 3 --no-cpu-baseline > $O/share_n$n.json 2> $O/share_n$n.err
  echo "share-gpu N=$n rc=$?" >> $O/summary.txt
done
