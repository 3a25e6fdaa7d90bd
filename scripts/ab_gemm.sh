#!/bin/bash
# A/B the GEMM microbenchmark between the in-tree library and another build
# (path relative to the repo root in $1), interleaved 3 times.
for i in 1 2 3; do
  python scripts/gemm_bench.py | sed "s/^{/{\"lib\":\"new\",/" >> gpurun_out/ab.jsonl
  DC_LIB_AB=$1 python scripts/gemm_bench.py | sed 's/^{/{"lib":"old",/' >> gpurun_out/ab.jsonl
done
