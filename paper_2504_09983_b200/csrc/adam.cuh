// The Adam update of one fp32 element (Adam; reading D18 of
// DESIGN.md for the operand order), shared by every kernel that applies it:
// rs_adam (comm.cu), the fused dW epilogue and the GEMM side job
// (gemm_sm100.cu).  Correctly rounded fp32 intrinsics, no FMA contraction:
//   g = sum * (1/(N n))          (n accumulated micro-steps; sum includes the
//                                 accumulated fp32 shard: acc + rs, reading D27)
//   m = m + (1-b1) * (g - m)
//   v = (b2 * v) + ((1-b2) * g) * g
//   d = sqrt(v) / c + eps
//   p = p + ((-s) * m) / d
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

namespace dc {

struct AdamScalars {
  float w1, w2, b2, neg_s, c, eps, invN;
  float rc;            // RN(1 / c), once per thread
};

__device__ __forceinline__ AdamScalars adam_scalars(float w1, float w2, float b2, float neg_s, float c, float eps,
                                                    float invN) {
  return AdamScalars{w1, w2, b2, neg_s, c, eps, invN, __frcp_rn(c)};
}

// SCALE = false: the caller knows invN == 1 (N = 1, one micro-step), where
// g * 1 == g exactly, so the multiply is dropped (the bulk N = 1 update)
template <bool SCALE = true>
__device__ __forceinline__ void adam_elem(float gsum, float& p, float& m, float& v, const AdamScalars& a) {
  const float g = SCALE ? __fmul_rn(gsum, a.invN) : gsum;
  m = __fadd_rn(m, __fmul_rn(a.w1, __fsub_rn(g, m)));
  v = __fadd_rn(__fmul_rn(a.b2, v), __fmul_rn(__fmul_rn(a.w2, g), g));
#ifndef DC_ADAM_DIV_RN
  // sqrt(v) / c with the step constant's reciprocal rc = RN(1/c) and two FMA
  // residual corrections (Markstein): equal to div.rn for every x in
  // [2^-75, 2^64], which holds every sqrt of a finite v >= 0 except 0, where
  // both give 0 (exhaustive check: profiles/r01g/adam_div/).  Three fewer
  // instructions than div.rn's fast path: at the power-capped in-step clock
  // (~1.43 GHz) the bulk rs_adam kernel's consumers are close to issue-bound,
  // and this takes rs 33.8 -> 32.7 ms per step (profiles/r02/adam_rcp/).
  // -DDC_ADAM_DIV_RN restores div.rn (bit-identical results).
  const float x = __fsqrt_rn(v), rc = a.rc;
  const float q0 = __fmul_rn(x, rc);
  const float q1 = __fmaf_rn(__fmaf_rn(-a.c, q0, x), rc, q0);
  const float d = __fadd_rn(__fmaf_rn(__fmaf_rn(-a.c, q1, x), rc, q1), a.eps);
#else
  const float d = __fadd_rn(__fdiv_rn(__fsqrt_rn(v), a.c), a.eps);
#endif
  p = __fadd_rn(p, __fdiv_rn(__fmul_rn(a.neg_s, m), d));
}

// L2 evict-first streaming accesses (the optimizer state is touched once per
// step; the GEMM operand tiles it runs beside live in L2)
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ld_stream(const void* ptr, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_stream(void* ptr, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(ptr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// One group of 8 consecutive shard elements, in two phases so a caller can
// keep several groups' loads in flight before any arithmetic (warps issue in
// order: the first dependent add would stall every later load):
//   load_group8:   fp32 master/m/v and the bf16 grads of `world` ranks
//   finish_group8: grads summed in ascending rank order from +0.0 (bf16 ->
//                  fp32), Adam on master/m/v, RNE bf16 shard, streaming stores
//   ACC:           the final micro-step of gradient accumulation adds the
//                  fp32 accumulated shard: g = acc + sum (one rounding)
template <int MAXQ>
struct Group8 {
  uint4 P[2], M[2], V[2], A[2], G[MAXQ];
};

template <int MAXQ, bool ACC = false>
__device__ __forceinline__ void load_group8(Group8<MAXQ>& x, const uint8_t* const* gptr, int world,
                                            const float* mst, const float* mm, const float* vv, uint64_t pol,
                                            const float* acc = nullptr) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    x.P[h] = ld_stream(mst + 4 * h, pol);
    x.M[h] = ld_stream(mm + 4 * h, pol);
    x.V[h] = ld_stream(vv + 4 * h, pol);
    if constexpr (ACC) x.A[h] = ld_stream(acc + 4 * h, pol);
  }
#pragma unroll
  for (int q = 0; q < MAXQ; ++q)
    if (q < world) x.G[q] = ld_stream(gptr[q], pol);
}

// sum over ranks in ascending order from +0.0 of the bf16 grads (fp32)
template <int MAXQ>
__device__ __forceinline__ void sum_ranks8(const uint4* G, int world, float (&g)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) g[j] = 0.0f;
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) {
    if (q < world) {
      float f[8];
      bf16x8_to_f32(G[q], f);
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = __fadd_rn(g[j], f[j]);
    }
  }
}

template <int MAXQ, bool ACC = false>
__device__ __forceinline__ void finish_group8(const Group8<MAXQ>& x, int world, float* mst, float* mm, float* vv,
                                              __nv_bfloat16* sh, const AdamScalars& a, uint64_t pol) {
  float g[8];
  sum_ranks8<MAXQ>(x.G, world, g);
  if constexpr (ACC) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float* af = reinterpret_cast<const float*>(&x.A[h]);
#pragma unroll
      for (int t = 0; t < 4; ++t) g[4 * h + t] = __fadd_rn(af[t], g[4 * h + t]);
    }
  }
  float pp[8], m8[8], v8[8];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float* pf = reinterpret_cast<const float*>(&x.P[h]);
    const float* mf = reinterpret_cast<const float*>(&x.M[h]);
    const float* vf = reinterpret_cast<const float*>(&x.V[h]);
#pragma unroll
    for (int t = 0; t < 4; ++t) { pp[4 * h + t] = pf[t]; m8[4 * h + t] = mf[t]; v8[4 * h + t] = vf[t]; }
  }
  uint4 out;
  __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
  for (int j = 0; j < 8; ++j) adam_elem(g[j], pp[j], m8[j], v8[j], a);
#pragma unroll
  for (int t = 0; t < 4; ++t) o2[t] = __floats2bfloat162_rn(pp[2 * t], pp[2 * t + 1]);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    st_stream(mst + 4 * h, *reinterpret_cast<const uint4*>(&pp[4 * h]), pol);
    st_stream(mm + 4 * h, *reinterpret_cast<const uint4*>(&m8[4 * h]), pol);
    st_stream(vv + 4 * h, *reinterpret_cast<const uint4*>(&v8[4 * h]), pol);
  }
  st_stream(sh, out, pol);
}

}  // namespace dc
