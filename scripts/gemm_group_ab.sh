# GEMM tile-order A/B: heuristic grouping (default) vs none (DC_GEMM_GROUP_M=0) — DRAM bytes of the first
# 16 GEMM launches of a 2-layer bench (ncu), alternating default bench lines, then the GPU suite
mkdir -p gpurun_out/gg2
for g in -1 0; do
  DC_GEMM_GROUP_M=$g timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:gemm2 -s 0 -c 16 --csv --log-file gpurun_out/gg2/dram_g$g.csv \
    python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
k=0
for g in -1 0 -1 0 -1 0; do
  k=$((k+1))
  DC_GEMM_GROUP_M=$g timeout 600 python bench.py --no-cpu-baseline 2> /dev/null | tail -1 > gpurun_out/gg2/bench_${k}_g$g.json
done
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/gg2/tests.log 2>&1
