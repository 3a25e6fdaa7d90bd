# GA accumulate modes at N = 1: two groups per thread (default) vs one (DC_RS_UNR=1), --micro 4, alternating
mkdir -p gpurun_out/rsga
k=0
for v in "" "-DDC_RS_UNR=1" "" "-DDC_RS_UNR=1"; do
  k=$((k+1))
  touch paper_2504_09983_b200/csrc/comm.cu
  DC_NVCC_EXTRA="$v" python -c "from paper_2504_09983_b200 import build as b; b.build()" > /dev/null
  timeout 900 python bench.py --no-cpu-baseline --micro 4 2> /dev/null | tail -1 > gpurun_out/rsga/$k.json
done
touch paper_2504_09983_b200/csrc/comm.cu
python -c "from paper_2504_09983_b200 import build as b; b.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_accum.py -q -m gpu > gpurun_out/rsga/tests.log 2>&1
