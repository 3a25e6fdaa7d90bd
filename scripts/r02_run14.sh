#!/bin/bash
# half-width tail units: GEMM parity, then in-step A/B (alternating)
O=gpurun_out/r02run14; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -k gemm -q -p no:cacheprovider > $O/gemm_tests.log 2>&1
echo "gemm tests rc=$? $(tail -1 $O/gemm_tests.log)" > $O/summary.txt
for rep in 1 2 3; do
  for ht in 0 1; do
    DC_GEMM_HALF_TAIL=$ht timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/ht${ht}_$rep.json 2> $O/ht${ht}_$rep.err
  done
done
