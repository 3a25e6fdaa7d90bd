"""One dc_gemm shape launched `reps` times (for ncu captures and A/B runs).
Usage: gemm_one.py M N K kernel reps [layout] [stream_k]
layout: fwd (A [M][K], B [N][K]), dx (A [M][K], B [K][N]), dw (A [K][M], B [K][N])"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_09983_b200 import dc  # noqa: E402

M, N, K, kern, reps = (int(a) for a in sys.argv[1:6])
layout = sys.argv[6] if len(sys.argv) > 6 else "fwd"
sk = int(sys.argv[7]) if len(sys.argv) > 7 else 1
dev = torch.device("cuda", 0)
a_mn = layout == "dw"
b_mn = layout in ("dx", "dw")
A = (torch.randn(*((K, M) if a_mn else (M, K)), device=dev) * 0.5).to(torch.bfloat16)
B = (torch.randn(*((K, N) if b_mn else (N, K)), device=dev) * 0.5).to(torch.bfloat16)
Cm = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
g = dc.GemmArgs()
g.M, g.N, g.K = M, N, K
g.A, g.lda, g.a_mn_major = A.data_ptr(), (M if a_mn else K), int(a_mn)
g.n_bseg = 1
g.B[0], g.ldb[0], g.bseg_end[0] = B.data_ptr(), (N if b_mn else K), N // 256
g.b_mn_major = int(b_mn)
g.C, g.ldc, g.kernel = Cm.data_ptr(), N, kern
g.stream_k = sk
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
ref = (A.float().T if a_mn else A.float()) @ (B.float() if b_mn else B.float().T)
err = ((Cm.float() - ref).norm() / ref.norm()).item()
print("sk %d M %d N %d K %d kernel %d %s: %.4f ms %.1f TFLOP/s relerr %.2e" % (sk, M, N, K, kern, layout, ms,
                                                                      2 * M * N * K / ms / 1e9, err))
