#!/bin/bash
# fused AG with the warp-cooperative chunk watcher: tests + A/B
O=gpurun_out/r02run11; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused_ag.py tests/test_gpu_kernels.py -k "fused or ag_ or gemm" -q -p no:cacheprovider > $O/tests.log 2>&1
echo "tests rc=$? $(tail -1 $O/tests.log)" > $O/summary.txt
for rep in 1 2; do
for p in S0 PS; do
  for f in 0 1; do
    DC_SPIN_MS=5000 timeout 300 python scripts/fused_ab.py --world 2 --layers 2 --batch 1 --steps 5 --fused $f --passes $p \
        >> $O/fused_ab.jsonl 2>> $O/fused_ab_${p}_$f.err
    echo "fused_ab $p fused=$f rc=$?" >> $O/summary.txt
  done
done
done
