#!/bin/bash
# (1) graph mode at N > 1 with every stream on ONE hardware connection: if the
#     virtual-rank stalls come from queue sharing between ranks, this makes
#     them near-certain (bounded waits: DC_SPIN_MS); (2) config-5 proxy: 70B
#     layers at N = 1 sized so the adaptive offload is small (the hideable
#     regime of N = 2, L = 24); (3) launch list of the default command.
mkdir -p gpurun_out/r02run4
R=gpurun_out/r02run4/summary.txt
: > $R
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02run4/bench.json 2> gpurun_out/r02run4/bench.err
timeout 900 python -m pytest tests/test_gpu_fused_ag.py -q -p no:cacheprovider > gpurun_out/r02run4/fused_ag.log 2>&1
echo "fused_ag + jitter tests rc=$? $(tail -1 gpurun_out/r02run4/fused_ag.log)" >> $R
timeout 1800 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/r02run4/racecheck_smoke.txt 2>&1
echo "racecheck rc=$? $(tail -2 gpurun_out/r02run4/racecheck_smoke.txt | tr '\n' ' ')" >> $R
for c in 1 32; do
  for i in 1 2 3; do
    CUDA_DEVICE_MAX_CONNECTIONS=$c DC_SPIN_MS=5000 DC_TEST_GRAPH_N=1 timeout 600 python -m pytest tests/test_gpu_graph.py \
        -k virtual_ranks -q -p no:cacheprovider > gpurun_out/r02run4/graph_c${c}_$i.log 2>&1
    echo "connections=$c run $i rc=$? $(tail -1 gpurun_out/r02run4/graph_c${c}_$i.log)" >> $R
    grep -o "timed out.*" gpurun_out/r02run4/graph_c${c}_$i.log | head -2 >> $R
  done
done
for L in 11 12; do
  timeout 900 python bench.py --offload --model llama3-70b --layers $L --batch 1 --steps 3 --warmup 3 --no-cpu-baseline \
      > gpurun_out/r02run4/offload_70b_L$L.json 2> gpurun_out/r02run4/offload_70b_L$L.err
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02run4/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02run4/ncu_bench.out 2>&1
