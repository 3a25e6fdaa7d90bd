mkdir -p gpurun_out/r02c
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "rs_adam" -p no:cacheprovider > gpurun_out/r02c/pytest_rs.txt 2>&1
echo "rc=$?" >> gpurun_out/r02c/pytest_rs.txt
timeout 300 python scripts/rs_bench.py 1 12 > gpurun_out/r02c/rs_bench_n1.json 2>&1
for b in 1 0 1 0; do
  DC_RS_BULK=$b timeout 900 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/r02c/bench_bulk$b.$RANDOM.json 2>/dev/null
done
