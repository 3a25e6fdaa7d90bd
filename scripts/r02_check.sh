# round-2 GPU check: tests, smoke (plain and under ncu), share-GPU loop, default bench
mkdir -p gpurun_out/r02a
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02a/build.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02a/pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02a/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a/smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/r02a/smoke.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all --csv \
  --log-file gpurun_out/r02a/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a/smoke_ncu.txt 2>&1
echo "ncu smoke rc=$?" >> gpurun_out/r02a/smoke_ncu.txt
bash scripts/share_loop.sh 8
cp gpurun_out/sl/res.txt gpurun_out/r02a/share_loop.txt
timeout 900 python bench.py > gpurun_out/r02a/bench.json 2> gpurun_out/r02a/bench.err
