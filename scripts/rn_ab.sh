mkdir -p gpurun_out/rn2
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_moe.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -1 > gpurun_out/rn2/tests.txt
for f in 0 2; do
  DC_RMSNORM_BWD=$f timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:rmsnorm_bwd|colsum" -s 24 -c 9 --csv python scripts/op_times.py LLAMA3_8B 2 2 > gpurun_out/rn2/ncu_$f.csv 2>&1
  for i in 1 2; do DC_RMSNORM_BWD=$f timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/rn2/b${f}_$i.json 2>&1; done
done
