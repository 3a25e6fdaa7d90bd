#!/bin/bash
# fused AG -> GEMM + NVLS gating tests, then the suites they touch
mkdir -p gpurun_out/r02fused
timeout 900 python -m pytest tests/test_gpu_fused_ag.py tests/test_gpu_nvls.py -x -q -p no:cacheprovider > gpurun_out/r02fused/new.log 2>&1
echo "rc=$?" >> gpurun_out/r02fused/new.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02fused/all.log 2>&1
echo "rc=$?" >> gpurun_out/r02fused/all.log
