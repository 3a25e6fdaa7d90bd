// SiLU(gate) * up and its backward in fp32, shared by the stand-alone glue
// kernels (glue.cu) and the GEMM epilogues that fuse them (gemm_sm100.cu), so
// the fused and unfused paths are bit-identical.  Inputs are the bf16-stored
// values (as fp32), outputs are rounded to bf16: the sigmoid uses the hardware
// exp2 / reciprocal approximations (relative error ~1e-6, 2^-8 is the bf16 step),
// the products explicit IEEE roundings (no FMA contraction).  These kernels are
// ALU-bound as much as HBM-bound with the IEEE expf / division.
#pragma once
#include <cuda_runtime.h>

namespace dc {

__device__ __forceinline__ float sigmoid_rn(float z) { return __fdividef(1.0f, __fadd_rn(1.0f, __expf(-z))); }

// act = (g * sigmoid(g)) * u
__device__ __forceinline__ float silu_mul(float g, float u) { return __fmul_rn(__fmul_rn(g, sigmoid_rn(g)), u); }

// d_up = da * (g s) ; d_gate = (da u) * (s (1 + g (1 - s)))
__device__ __forceinline__ void silu_mul_bwd(float da, float g, float u, float& dg, float& du) {
  const float s = sigmoid_rn(g);
  du = __fmul_rn(da, __fmul_rn(g, s));
  dg = __fmul_rn(__fmul_rn(da, u), __fmul_rn(s, __fadd_rn(1.0f, __fmul_rn(g, __fsub_rn(1.0f, s)))));
}

}  // namespace dc
