# tall-grid group size (only GEMMs with m_tiles >= 2 n_tiles are grouped): 2 vs 8, alternating builds
mkdir -p gpurun_out/gg6
k=0
for g in 2 8 2 8; do
  k=$((k+1))
  touch paper_2504_09983_b200/csrc/gemm_sm100.cu
  DC_NVCC_EXTRA="-DDC_GEMM_GROUP_DEFAULT=$g" python -c "from paper_2504_09983_b200 import build as b; b.build()" > /dev/null 2>&1
  timeout 600 python bench.py --no-cpu-baseline 2> /dev/null | tail -1 > gpurun_out/gg6/bench_${k}_g$g.json
done
touch paper_2504_09983_b200/csrc/gemm_sm100.cu
python -c "from paper_2504_09983_b200 import build as b; b.build()" > /dev/null 2>&1
