#!/bin/bash
# final build (reciprocal Adam division, preload fix): GPU suite, smoke, default bench x2, reference arm, launch list
O=gpurun_out/r02s3final2; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "gpu suite rc=$? $(grep -E 'passed|failed' $O/pytest_gpu.log | tail -1)" > $O/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$? $(tail -1 $O/smoke.log)" >> $O/summary.txt
for rep in 1 2; do
  timeout 900 python bench.py > $O/bench_default_$rep.json 2> $O/bench_default_$rep.err
  echo "bench $rep rc=$?" >> $O/summary.txt
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
echo "reference rc=$?" >> $O/summary.txt
timeout 900 python bench.py --model llama3-70b --steps 5 --no-cpu-baseline > $O/llama70b_L8.json 2> $O/llama70b_L8.err
timeout 900 python bench.py --model mixtral-8x7b --batch 2 --steps 5 --no-cpu-baseline > $O/mixtral_b2.json 2> $O/mixtral_b2.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_bench.out 2>&1
echo "launch list rc=$?" >> $O/summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rs_adam_bulk -s 8 -c 1 \
    -o $O/rs_adam python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_rs.out 2>&1
echo "ncu rs rc=$?" >> $O/summary.txt
