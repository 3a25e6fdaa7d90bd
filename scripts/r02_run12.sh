#!/bin/bash
# stream-K for the K = 4096 / 6144 GEMMs (o_proj, qkv and their dX) in-step A/B, alternating
O=gpurun_out/r02run12; mkdir -p $O
for rep in 1 2 3; do
  for kb in 128 64; do
    DC_GEMM_SK_MINKB=$kb timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/sk${kb}_$rep.json 2> $O/sk${kb}_$rep.err
  done
done
