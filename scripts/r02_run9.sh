#!/bin/bash
# suite stability after the virtual-rank stream reduction (x2), fused AG A/B with issue-ordered GEMMs
O=gpurun_out/r02run9; mkdir -p $O
: > $O/summary.txt
for i in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_$i.log 2>&1
  echo "gpu suite $i rc=$? $(tail -1 $O/pytest_gpu_$i.log)" >> $O/summary.txt
done
for p in S0 PS; do
  for f in 0 1; do
    DC_SPIN_MS=5000 timeout 300 python scripts/fused_ab.py --world 2 --layers 2 --batch 1 --steps 5 --fused $f --passes $p \
        >> $O/fused_ab.jsonl 2>> $O/fused_ab_${p}_$f.err
    echo "fused_ab $p fused=$f rc=$?" >> $O/summary.txt
  done
done
