# rs_adam occupancy A/B: groups per thread (DC_RS_UNR) x min CTAs per SM (DC_RS_MINB) x grid,
# interleaved (box-to-box variance is larger than the effect; compare within one call)
mkdir -p gpurun_out/rsab4
k=0
for v in ${RSAB_VARIANTS:-"2 1 296" "1 1 296" "1 2 296" "1 4 296" "1 4 444" "2 1 296" "1 1 296" "1 2 296" "1 4 296" "1 4 444"}; do
  set -- $v
  k=$((k+1))
  touch paper_2504_09983_b200/csrc/comm.cu
  DC_NVCC_EXTRA="-DDC_RS_UNR=$1 -DDC_RS_MINB=$2" python -c "from paper_2504_09983_b200 import build as b; b.build()" > /dev/null
  for rep in 1 2; do
    DC_RS_CTAS=$3 DCOPT_RS_OVERLAP=0 timeout 200 python scripts/op_times.py LLAMA3_8B 4 2 > gpurun_out/rsab4/${k}_u$1_b$2_c$3_r${rep}.txt 2>&1
  done
done
touch paper_2504_09983_b200/csrc/comm.cu
python -c "from paper_2504_09983_b200 import build as b; b.build()" > /dev/null
