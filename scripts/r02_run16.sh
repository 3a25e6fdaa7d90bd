#!/bin/bash
# half-width tail units on the forward GEMMs only: in-step A/B, alternating
O=gpurun_out/r02run16; mkdir -p $O
for rep in 1 2 3; do
  for ht in 0 1; do
    DC_GEMM_HALF_TAIL=$ht timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/ht${ht}_$rep.json 2> $O/ht${ht}_$rep.err
  done
done
