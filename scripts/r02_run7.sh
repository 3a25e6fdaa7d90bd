#!/bin/bash
# after: chunk-watcher warp (fused AG -> GEMM), CW kernel instantiation, deferred state write-back join
O=gpurun_out/r02run7; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "gpu suite rc=$? $(tail -1 $O/pytest_gpu.log)" > $O/summary.txt
for p in S0 PS; do
  for f in 0 1; do
    DC_SPIN_MS=5000 timeout 300 python scripts/fused_ab.py --world 2 --layers 2 --batch 1 --steps 5 --fused $f --passes $p \
        >> $O/fused_ab.jsonl 2>> $O/fused_ab_${p}_$f.err
    echo "fused_ab $p fused=$f rc=$?" >> $O/summary.txt
  done
done
for rep in 1 2; do
  (cd abtree && timeout 600 python bench.py --no-cpu-baseline --steps 10) > $O/old_$rep.json 2> $O/old_$rep.err
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/new_$rep.json 2> $O/new_$rep.err
done
for L in 13 14; do
  timeout 900 python bench.py --offload --model llama3-70b --layers $L --batch 1 --steps 3 --warmup 3 --no-cpu-baseline \
      > $O/offload_70b_L$L.json 2> $O/offload_70b_L$L.err
  echo "offload L=$L rc=$?" >> $O/summary.txt
done
