"""Microbenchmark of dc_gemm on the Llama-3-8B layer shapes (T tokens):
forward (K-major x K-major), dX (K-major x MN-major, K-split) and dW
(MN-major x MN-major), for the 1-CTA and CTA-pair kernels, plus torch.matmul
(cuBLAS) as a same-box comparator.  CUDA events, warm-up, median of reps.
Prints one JSON line per case."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_09983_b200 import dc  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
H, F, QKV = 4096, 14336, 6144
dev = torch.device("cuda", 0)


def rnd(*shape):
    return (torch.randn(*shape, device=dev) * 0.5).to(torch.bfloat16)


def run(name, M, N, K, A, lda, a_mn, Bs, ldbs, ends, b_mn, split_k, kernel, reps=20):
    Cm = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    g = dc.GemmArgs()
    g.M, g.N, g.K = M, N, K
    g.A, g.lda, g.a_mn_major = A.data_ptr(), lda, a_mn
    g.n_bseg = len(Bs)
    for i, (b, l, e) in enumerate(zip(Bs, ldbs, ends)):
        g.B[i], g.ldb[i], g.bseg_end[i] = b.data_ptr(), l, e
    g.b_mn_major, g.b_split_k = b_mn, split_k
    g.C, g.ldc, g.kernel = Cm.data_ptr(), N, kernel
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        dc.check(dc.lib.dc_gemm(C.byref(g), st))
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dc.check(dc.lib.dc_gemm(C.byref(g), st))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    return {"case": name, "kernel": {1: "cta1", 2: "pair"}[kernel], "M": M, "N": N, "K": K, "ms": ms,
            "tflops": 2.0 * M * N * K / (ms * 1e-3) / 1e12}


def torch_ref(name, M, N, K, reps=20):
    a, b = rnd(M, K), rnd(K, N)
    for _ in range(3):
        torch.matmul(a, b)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    return {"case": name, "kernel": "cublas", "M": M, "N": N, "K": K, "ms": ms,
            "tflops": 2.0 * M * N * K / (ms * 1e-3) / 1e12}


x = rnd(T, H)
wg, wu, wd = rnd(F, H), rnd(F, H), rnd(H, F)
gu = rnd(T, 2 * F)
act = rnd(T, F)
dy = rnd(T, H)
cases = []
for kern in (1, 2):
    cases.append(run("gate_up fwd", T, 2 * F, H, x, H, 0, [wg, wu], [H, H], [F // 256, 2 * F // 256], 0, 0, kern))
    cases.append(run("down fwd", T, H, F, act, F, 0, [wd], [F], [H // 256], 0, 0, kern))
    cases.append(run("o fwd", T, H, H, x, H, 0, [wd[:, :H].contiguous()], [H], [H // 256], 0, 0, kern))
    cases.append(run("gate_up dX", T, H, 2 * F, gu, 2 * F, 0, [wg, wu], [H, H], [F // 64, 2 * F // 64], 1, 1, kern))
    cases.append(run("down dX", T, F, H, dy, H, 0, [wd], [F], [F // 256], 1, 0, kern))
    cases.append(run("gate dW", F, H, T, gu, 2 * F, 1, [x], [H], [H // 256], 1, 0, kern))
    cases.append(run("down dW", H, F, T, dy, H, 1, [act], [F], [F // 256], 1, 0, kern))
cases.append(torch_ref("gate_up fwd", T, 2 * F, H))
cases.append(torch_ref("o fwd", T, H, H))
for c in cases:
    print(json.dumps(c))
