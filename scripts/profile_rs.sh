mkdir -p gpurun_out/prof2
timeout 900 python bench.py > gpurun_out/prof2/bench_default.json 2> gpurun_out/prof2/bench_default.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof2/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rs_adam -s 12 -c 1 -o gpurun_out/prof2/rs_adam python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/prof2
