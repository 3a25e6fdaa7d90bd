#!/bin/bash
# Round profile artifacts (run under gpurun; outputs in gpurun_out/prof/):
#  launches.csv  - ncu launch list (gpu__time_duration.sum, clock-control none)
#                  of a short 2-layer bench run (cold-cache, serialised: SHARES)
#  gemm2.ncu-rep - ncu --set full of 6 backward pair-GEMM launches
#  rs_adam.ncu-rep - ncu --set full of one rs_adam launch
set -x
mkdir -p gpurun_out/prof
B="python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm2 -s 40 -c 6 -o gpurun_out/prof/gemm2 \
    python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rs_adam -s 12 -c 1 -o gpurun_out/prof/rs_adam \
    python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/prof
