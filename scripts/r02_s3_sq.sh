#!/bin/bash
# tile groups for square long-K GEMMs (DC_GEMM_GROUP_SQ = 0 / 4 / 8): in-step A/B, ncu DRAM + time per launch
O=gpurun_out/r02s3sq; mkdir -p $O
for rep in 1 2; do
  for g in 0 4 8; do
    DC_GEMM_GROUP_SQ=$g timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/sq${g}_$rep.json 2> $O/sq${g}_$rep.err
  done
done
for g in 0 4 8; do
  DC_GEMM_GROUP_SQ=$g timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:gemm2 -c 16 --csv --log-file $O/ncu_sq$g.csv \
    python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
done
DC_GEMM_GROUP_SQ=8 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "gemm or fullsize" > $O/pytest_sq8.log 2>&1
echo "sq8 tests rc=$? $(tail -1 $O/pytest_sq8.log)" > $O/summary.txt
