mkdir -p gpurun_out/gg3
for g in -1 0 -1 0; do
  k=$((k+1))
  DC_GEMM_GROUP_M=$g timeout 600 python bench.py --no-cpu-baseline --model mixtral-8x7b 2> /dev/null | tail -1 > gpurun_out/gg3/mix_${k}_g$g.json
  DC_GEMM_GROUP_M=$g timeout 600 python bench.py --no-cpu-baseline --model llama3-70b 2> /dev/null | tail -1 > gpurun_out/gg3/l70_${k}_g$g.json
done
