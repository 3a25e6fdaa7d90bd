#!/bin/bash
# SwiGLU kernels with two chunks per thread + resident-sized grids (this tree) vs HEAD~ (abtree/): A/B, ncu
O=gpurun_out/r02s3act; mkdir -p $O
for rep in 1 2 3; do
  (cd abtree && timeout 600 python bench.py --no-cpu-baseline --steps 10) > $O/prev_$rep.json 2> $O/prev_$rep.err
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/new_$rep.json 2> $O/new_$rep.err
done
for t in . abtree; do
  n=$( [ "$t" = . ] && echo new || echo prev )
  (cd $t && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"act_|attn_mix" -s 40 -c 24 --csv --log-file ../$O/glue_$n.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1)
done
cp abtree/$O/glue_prev.csv $O/ 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py tests/test_gpu_moe.py -q -p no:cacheprovider > $O/pytest_sub.log 2>&1
echo "subset rc=$? $(grep -E 'passed|failed' $O/pytest_sub.log | tail -1)" > $O/summary.txt
