#!/bin/bash
# stream-K on/off on the Llama-3-8B layer GEMM shapes (T = 4096)
for sk in 0 1 0 1; do
  python scripts/gemm_one.py 4096 4096 4096 2 30 fwd $sk
  python scripts/gemm_one.py 4096 4096 14336 2 20 fwd $sk
  python scripts/gemm_one.py 4096 6144 4096 2 30 fwd $sk
  python scripts/gemm_one.py 4096 4096 28672 2 10 dx $sk
  python scripts/gemm_one.py 4096 14336 4096 2 20 dx $sk
  python scripts/gemm_one.py 4096 4096 4096 2 30 dw $sk
  python scripts/gemm_one.py 14336 4096 4096 2 20 dw $sk
  python scripts/gemm_one.py 4096 28672 4096 2 10 fwd $sk
done
