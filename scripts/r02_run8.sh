#!/bin/bash
# S0 + fused_ag diagnosis (fail-fast chunk waits), bulk push v2 sweep + ncu, side-job test
O=gpurun_out/r02run8; mkdir -p $O
DC_SPIN_MS=4000 timeout 300 python scripts/fused_ab.py --world 2 --layers 2 --batch 1 --steps 2 --fused 1 --passes S0 \
    > $O/fused_s0.jsonl 2> $O/fused_s0.err
echo "fused S0 rc=$?" > $O/summary.txt
timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_fused_ag.py -q -p no:cacheprovider > $O/tests.log 2>&1
echo "model + fused tests rc=$? $(tail -1 $O/tests.log)" >> $O/summary.txt
timeout 1500 python scripts/ag_sweep.py --worlds 2,8 --modes sm,bulk --max-log2 31 --steps 5 --out $O/ag_sweep_bulk.json > $O/ag_sweep.txt 2>&1
echo "sweep rc=$?" >> $O/summary.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ag_push -c 4 -o $O/ag_push_n8_bulk \
    python scripts/ag_sweep.py --ncu-push 8 --max-log2 30 --modes bulk > $O/ncu_ag_bulk.txt 2>&1
echo "ncu bulk rc=$?" >> $O/summary.txt
