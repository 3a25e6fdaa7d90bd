#!/bin/bash
mkdir -p gpurun_out/r02run3
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02run3/bench.json 2> gpurun_out/r02run3/bench.err
timeout 600 python bench.py --no-cpu-baseline --steps 5 --tc-table profiles/r02/collectives/ag_sweep.json:8:sm \
    --profile-json gpurun_out/r02run3/whatif_plan.json > gpurun_out/r02run3/bench_whatif.json 2> gpurun_out/r02run3/bench_whatif.err
bash scripts/r02_stalls.sh 10 5
