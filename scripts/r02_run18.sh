#!/bin/bash
# T_c(V) sweep with a start gate (no host enqueue skew in small gathers)
O=gpurun_out/r02run18; mkdir -p $O
timeout 1800 python scripts/ag_sweep.py --worlds 2,4,8 --modes sm,ce --max-log2 31 --steps 5 --out $O/ag_sweep_gated.json > $O/ag_sweep.txt 2>&1
echo "sweep rc=$?" >> $O/ag_sweep.txt
