mkdir -p gpurun_out/r02b
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "rs_adam" -p no:cacheprovider > gpurun_out/r02b/pytest_rs.txt 2>&1
echo "rc=$?" >> gpurun_out/r02b/pytest_rs.txt
timeout 600 python -m pytest tests/test_gpu_moe.py -q -m gpu -p no:cacheprovider > gpurun_out/r02b/pytest_moe.txt 2>&1
echo "rc=$?" >> gpurun_out/r02b/pytest_moe.txt
timeout 300 python scripts/rs_bench.py 1 12 > gpurun_out/r02b/rs_bench_n1.json 2>&1
timeout 300 python scripts/rs_bench.py 2 8 > gpurun_out/r02b/rs_bench_n2.json 2>&1
for b in 1 0 1 0; do
  DC_RS_BULK=$b timeout 900 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/r02b/bench_bulk$b.$RANDOM.json 2>/dev/null
done
