#!/bin/bash
O=gpurun_out/r02run10; mkdir -p $O
timeout 900 python scripts/ag_sweep.py --worlds 2 --modes sm,chunked --max-log2 30 --steps 5 --out $O/ag_sweep_chunked.json > $O/ag_sweep.txt 2>&1
python scripts/hbm_patterns.py > $O/hbm_patterns.json 2>&1
