mkdir -p gpurun_out/rsn1
for v in 1 2 1 2; do
  touch paper_2504_09983_b200/csrc/comm.cu
  DC_NVCC_EXTRA="-DDC_RS_UNR_N1=$v" python -c "from paper_2504_09983_b200 import build as b; b.build()" > /dev/null
  k=$((k+1))
  timeout 600 python bench.py > gpurun_out/rsn1/bench_${k}_u$v.json 2> gpurun_out/rsn1/bench_${k}_u$v.err
done
touch paper_2504_09983_b200/csrc/comm.cu
python -c "from paper_2504_09983_b200 import build as b; b.build()" > /dev/null
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/rsn1/tests.log 2>&1
