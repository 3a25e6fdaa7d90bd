# rs_adam software pipeline A/B (DC_RS_PIPE): op times of Llama-3-8B L = 4, b = 2, rs in stream order
mkdir -p gpurun_out/rsab3
for pp in 0 1 2; do
  touch paper_2504_09983_b200/csrc/comm.cu
  DC_NVCC_EXTRA="-DDC_RS_PIPE=$pp" python -c "from paper_2504_09983_b200 import build as b; b.build()" > /dev/null
  for ctas in 296 148; do
    for rep in 1 2; do
      DC_RS_CTAS=$ctas DCOPT_RS_OVERLAP=0 timeout 200 python scripts/op_times.py LLAMA3_8B 4 2 > gpurun_out/rsab3/p${pp}_c${ctas}_r${rep}.txt 2>&1
    done
  done
done
touch paper_2504_09983_b200/csrc/comm.cu
python -c "from paper_2504_09983_b200 import build as b; b.build()" > /dev/null
