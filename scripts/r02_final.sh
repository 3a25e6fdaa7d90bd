#!/bin/bash
# round-2 final-state evidence: GPU suite, smoke, default bench (+ reference arm), model lines, launch list
O=gpurun_out/r02final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "gpu suite rc=$? $(tail -1 $O/pytest_gpu.log)" > $O/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$? $(tail -1 $O/smoke.log)" >> $O/summary.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
echo "bench rc=$?" >> $O/summary.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
echo "reference rc=$?" >> $O/summary.txt
for b in 1 2 4; do
  timeout 900 python bench.py --model mixtral-8x7b --batch $b --steps 5 --no-cpu-baseline > $O/mixtral_b$b.json 2> $O/mixtral_b$b.err
done
timeout 900 python bench.py --model llama3-70b --steps 5 --no-cpu-baseline > $O/llama70b_L8.json 2> $O/llama70b_L8.err
timeout 900 python bench.py --micro 4 --steps 5 --no-cpu-baseline > $O/llama8b_ga4.json 2> $O/llama8b_ga4.err
timeout 900 python bench.py --checkpoint --steps 5 --no-cpu-baseline > $O/llama8b_ckpt.json 2> $O/llama8b_ckpt.err
timeout 900 python bench.py --offload --model llama3-70b --layers 16 --batch 1 --steps 3 --warmup 3 --no-cpu-baseline \
    > $O/offload_70b_L16.json 2> $O/offload_70b_L16.err
echo "lines done" >> $O/summary.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_bench.out 2>&1
echo "launch list rc=$?" >> $O/summary.txt
