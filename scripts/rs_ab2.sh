mkdir -p gpurun_out/rsab2
for pf in 0 1 2; do
  touch paper_2504_09983_b200/csrc/comm.cu
  DC_NVCC_EXTRA="-DDC_RS_PREFETCH=$pf" python -c "from paper_2504_09983_b200 import build as b; b.build()"
  for th in 256; do
    DC_RS_THREADS=$th DCOPT_RS_OVERLAP=0 timeout 200 python scripts/op_times.py LLAMA3_8B 4 2 > gpurun_out/rsab2/pf${pf}_t${th}.txt 2>&1
  done
done
