# Final-state artifacts: default bench line, ncu launch list of the default command (shares)
mkdir -p gpurun_out/pf
timeout 900 python bench.py > gpurun_out/pf/bench_default.json 2> gpurun_out/pf/bench_default.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pf/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
