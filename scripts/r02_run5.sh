#!/bin/bash
# (1) same-box A/B: the round-start build (abtree/, commit 60dda63) vs this tree, alternating;
# (2) fused all-gather -> GEMM A/B at 2 virtual ranks; (3) SwiGLU forward epilogue A/B
mkdir -p gpurun_out/r02run5
for rep in 1 2; do
  (cd abtree && timeout 600 python bench.py --no-cpu-baseline --steps 10) > gpurun_out/r02run5/old_$rep.json 2> gpurun_out/r02run5/old_$rep.err
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/r02run5/new_$rep.json 2> gpurun_out/r02run5/new_$rep.err
done
for rep in 1 2; do
  for p in S0 PS; do
    for f in 0 1; do
      timeout 600 python scripts/fused_ab.py --world 2 --layers 4 --batch 1 --steps 5 --fused $f --passes $p \
          >> gpurun_out/r02run5/fused_ab.jsonl 2>> gpurun_out/r02run5/fused_ab.err
    done
  done
done
for rep in 1 2; do
  for fa in 0 1; do
    DC_FUSE_ACT=$fa timeout 600 python bench.py --no-cpu-baseline --steps 10 \
        > gpurun_out/r02run5/bench_fa${fa}_$rep.json 2> gpurun_out/r02run5/bench_fa${fa}_$rep.err
  done
done
