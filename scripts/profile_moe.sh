#!/bin/bash
# r01g profile artifacts (run under gpurun; outputs in gpurun_out/prof_g/):
#  launches.csv     - launch list of a 2-layer Llama-3-8B-shaped bench run
#  mix_launches.csv - launch list of a 2-layer Mixtral-shaped bench run
#  moe.ncu-rep      - ncu --set full of the MoE glue kernels (router, gather, combine, backward)
#  expgemm.ncu-rep  - ncu --set full of 3 expert GEMMs (gate|up fwd, down fwd, gate|up dX)
#  glu.ncu-rep      - ncu --set full of the GLU-epilogue gate|up GEMM (DC_FUSE_ACT=1)
#  rs_adam_mix.ncu-rep - one Mixtral-layer rs_adam (1.45 G elements)
set -x
O=gpurun_out/prof_g
mkdir -p $O
B="python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu-baseline"
M="python bench.py --model mixtral-8x7b --layers 2 --steps 1 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/mix_launches.csv $M > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:moe -s 60 -c 6 -o $O/moe $M > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm2 -s 300 -c 3 -o $O/expgemm $M > /dev/null 2>&1
DC_FUSE_ACT=1 ncu --set full --clock-control none --import-source on -k "regex:gemm2.*6, 2>" -s 20 -c 2 -o $O/glu $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rs_adam -s 12 -c 1 -o $O/rs_adam_mix $M > /dev/null 2>&1
ls -la $O
