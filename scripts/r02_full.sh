#!/bin/bash
# round-2 checkpoint: GPU suite + default bench + smoke
set -x
mkdir -p gpurun_out/r02full
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02full/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02full/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02full/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02full/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r02full/bench.json 2> gpurun_out/r02full/bench.err
DC_RMSNORM_TWO_PASS=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02full/bench_rn2.json 2> gpurun_out/r02full/bench_rn2.err
