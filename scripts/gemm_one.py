"""One dc_gemm shape (forward layout: A [M][K], B [N][K]) launched `reps`
times — for ncu captures.  Usage: gemm_one.py M N K kernel reps"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_09983_b200 import dc  # noqa: E402

M, N, K, kern, reps = (int(a) for a in sys.argv[1:6])
dev = torch.device("cuda", 0)
A = (torch.randn(M, K, device=dev) * 0.5).to(torch.bfloat16)
B = (torch.randn(N, K, device=dev) * 0.5).to(torch.bfloat16)
Cm = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
g = dc.GemmArgs()
g.M, g.N, g.K = M, N, K
g.A, g.lda, g.a_mn_major = A.data_ptr(), K, 0
g.n_bseg = 1
g.B[0], g.ldb[0], g.bseg_end[0] = B.data_ptr(), K, N // 256
g.C, g.ldc, g.kernel = Cm.data_ptr(), N, kern
st = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    dc.check(dc.lib.dc_gemm(C.byref(g), st))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    dc.check(dc.lib.dc_gemm(C.byref(g), st))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print("M %d N %d K %d kernel %d: %.4f ms %.1f TFLOP/s" % (M, N, K, kern, ms, 2 * M * N * K / ms / 1e9))
