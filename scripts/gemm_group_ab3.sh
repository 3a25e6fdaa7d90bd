mkdir -p gpurun_out/gg4
for g in 4 2; do
  DC_GEMM_GROUP_M=$g timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:gemm2 -s 0 -c 16 --csv --log-file gpurun_out/gg4/dram_g$g.csv \
    python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
