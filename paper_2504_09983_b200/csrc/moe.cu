// Glue kernels of the Mixtral-shaped MoE MLP (
// PAPER.md line 440 names Mixtral 8x7B): fixed balanced top-2 routing, token t
// -> experts e0 = t mod E and e1 = (t+1) mod E, gates = softmax of those two
// router logits.  Every expert gets R = 2T/E rows; expert e's rows are its
// tokens in ascending order, stored expert-major ([E][R][.]) so each expert's
// GEMM operands are contiguous.  All kernels HBM-bound, fp32 math, bf16
// storage, fixed-order reductions (deterministic run to run).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "dc_internal.h"

namespace dc {

namespace {
using bf16 = __nv_bfloat16;
using bf162 = __nv_bfloat162;

__device__ __forceinline__ void ld8(const bf16* p, float (&f)[8]) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const bf162* h = reinterpret_cast<const bf162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ void st8(bf16* p, const float (&f)[8]) {
  uint4 u;
  bf162* h = reinterpret_cast<bf162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Expert e's two token residues mod E, (lo, hi) with lo < hi: e-1 and e, or
// 0 and E-1 for e = 0.  Row j of expert e is token (j/2) E + (j odd ? hi : lo).
__device__ __forceinline__ int exp_tok(int e, int j, int E) {
  const int lo = e == 0 ? 0 : e - 1, hi = e == 0 ? E - 1 : e;
  return (j >> 1) * E + ((j & 1) ? hi : lo);
}
// Row of token t inside expert e's block (e must be one of t's two experts).
__device__ __forceinline__ int exp_row(int t, int e, int E) {
  const int hi = e == 0 ? E - 1 : e;
  return 2 * (t / E) + ((t % E) == hi ? 1 : 0);
}

constexpr int MAX_E = 8;
constexpr int WPB = 8;   // warps (tokens) per block of the per-token kernels

// router: l_e = <h2[t], Wr[e]> (fp32); g0 = 1 / (1 + exp(l1 - l0)), g1 = 1 / (1 + exp(l0 - l1))
__global__ void __launch_bounds__(WPB * 32) moe_router_fwd_kernel(const bf16* __restrict__ h2, const bf16* __restrict__ wr,
                                                                  float* __restrict__ g01, int T, int H, int E) {
  const int t = blockIdx.x * WPB + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (t >= T) return;
  float acc[MAX_E];
#pragma unroll
  for (int e = 0; e < MAX_E; ++e) acc[e] = 0.0f;
  for (int c = lane * 8; c < H; c += 256) {
    float x[8];
    ld8(h2 + (int64_t)t * H + c, x);
#pragma unroll
    for (int e = 0; e < MAX_E; ++e) {
      if (e < E) {
        float w[8];
        ld8(wr + (int64_t)e * H + c, w);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[e] = fmaf(x[i], w[i], acc[e]);
      }
    }
  }
  const int e0 = t % E, e1 = (e0 + 1) % E;
  float l0 = 0.0f, l1 = 0.0f;
#pragma unroll
  for (int e = 0; e < MAX_E; ++e) {
    const float s = warp_sum(acc[e]);
    if (e == e0) l0 = s;
    if (e == e1) l1 = s;
  }
  if (lane == 0) {
    g01[2 * t] = 1.0f / (1.0f + expf(l1 - l0));
    g01[2 * t + 1] = 1.0f / (1.0f + expf(l0 - l1));
  }
}

// X[e][j] = h2[token(e, j)]  (16-byte vectors)
__global__ void moe_gather_kernel(const bf16* __restrict__ h2, bf16* __restrict__ X, int T, int H, int E) {
  const int R = 2 * T / E, hv = H / 8;
  const int64_t n = (int64_t)E * R * hv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / hv;
    const int c = (int)(i % hv);
    const int e = (int)(row / R), j = (int)(row % R);
    reinterpret_cast<uint4*>(X)[i] = reinterpret_cast<const uint4*>(h2)[(int64_t)exp_tok(e, j, E) * hv + c];
  }
}

// y[t] = bf16(x2[t] + g0 O[e0][row] + g1 O[e1][row])
__global__ void moe_combine_kernel(const bf16* __restrict__ x2, const bf16* __restrict__ O, const float* __restrict__ g01,
                                   bf16* __restrict__ y, int T, int H, int E) {
  const int R = 2 * T / E, hv = H / 8;
  const int64_t n = (int64_t)T * hv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / hv), c = (int)(i % hv) * 8;
    const int e0 = t % E, e1 = (e0 + 1) % E;
    const float g0 = g01[2 * t], g1 = g01[2 * t + 1];
    float a[8], o0[8], o1[8];
    ld8(x2 + (int64_t)t * H + c, a);
    ld8(O + ((int64_t)e0 * R + exp_row(t, e0, E)) * H + c, o0);
    ld8(O + ((int64_t)e1 * R + exp_row(t, e1, E)) * H + c, o1);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = a[k] + g0 * o0[k] + g1 * o1[k];
    st8(y + (int64_t)t * H + c, a);
  }
}

// combine backward, one warp per token:
//   dO[e_k][row] = bf16(g_k dy[t]);  dg_k = <dy[t], O[e_k][row]>;
//   dl0 = g0 g1 (dg0 - dg1)  (softmax of two logits: dl1 = -dl0)
__global__ void __launch_bounds__(WPB * 32) moe_combine_bwd_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ O,
                                                                   const float* __restrict__ g01, bf16* __restrict__ dO,
                                                                   float* __restrict__ dl0, int T, int H, int E) {
  const int t = blockIdx.x * WPB + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (t >= T) return;
  const int R = 2 * T / E;
  const int e0 = t % E, e1 = (e0 + 1) % E;
  const int64_t r0 = ((int64_t)e0 * R + exp_row(t, e0, E)) * H, r1 = ((int64_t)e1 * R + exp_row(t, e1, E)) * H;
  const float g0 = g01[2 * t], g1 = g01[2 * t + 1];
  float d0 = 0.0f, d1 = 0.0f;
  for (int c = lane * 8; c < H; c += 256) {
    float d[8], o0[8], o1[8], w0[8], w1[8];
    ld8(dy + (int64_t)t * H + c, d);
    ld8(O + r0 + c, o0);
    ld8(O + r1 + c, o1);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      d0 = fmaf(d[k], o0[k], d0);
      d1 = fmaf(d[k], o1[k], d1);
      w0[k] = g0 * d[k];
      w1[k] = g1 * d[k];
    }
    st8(dO + r0 + c, w0);
    st8(dO + r1 + c, w1);
  }
  d0 = warp_sum(d0);
  d1 = warp_sum(d1);
  if (lane == 0) dl0[t] = g0 * g1 * (d0 - d1);
}

// dh2[t] = bf16(dX[e0][row] + dX[e1][row] + dl0 (Wr[e0] - Wr[e1]))
__global__ void moe_router_dx_kernel(const bf16* __restrict__ dX, const float* __restrict__ dl0,
                                     const bf16* __restrict__ wr, bf16* __restrict__ dh2, int T, int H, int E) {
  const int R = 2 * T / E, hv = H / 8;
  const int64_t n = (int64_t)T * hv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / hv), c = (int)(i % hv) * 8;
    const int e0 = t % E, e1 = (e0 + 1) % E;
    const float dl = dl0[t];
    float a[8], b[8], w0[8], w1[8];
    ld8(dX + ((int64_t)e0 * R + exp_row(t, e0, E)) * H + c, a);
    ld8(dX + ((int64_t)e1 * R + exp_row(t, e1, E)) * H + c, b);
    ld8(wr + (int64_t)e0 * H + c, w0);
    ld8(wr + (int64_t)e1 * H + c, w1);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = a[k] + b[k] + dl * (w0[k] - w1[k]);
    st8(dh2 + (int64_t)t * H + c, a);
  }
}

// router weight grad partials: P[blk][e][c] = sum over the block's rows t (in
// order) of dlog[t][e] h2[t][c], dlog[t][e0] = dl0, dlog[t][e1] = -dl0.  Each
// thread owns 2 columns and all E accumulators (fixed order, no atomics).
constexpr int RG_ROWS = 64;
__global__ void __launch_bounds__(256) moe_router_dw_kernel(const bf16* __restrict__ h2, const float* __restrict__ dl0,
                                                            float* __restrict__ part, int T, int H, int E) {
  const int c = (blockIdx.y * 256 + threadIdx.x) * 2;
  if (c >= H) return;
  float acc[MAX_E][2];
#pragma unroll
  for (int e = 0; e < MAX_E; ++e) acc[e][0] = acc[e][1] = 0.0f;
  const int r0 = blockIdx.x * RG_ROWS;
  for (int t = r0; t < r0 + RG_ROWS && t < T; ++t) {
    const float2 x = __bfloat1622float2(*reinterpret_cast<const bf162*>(h2 + (int64_t)t * H + c));
    const float dl = dl0[t];
    const int e0 = t % E, e1 = (e0 + 1) % E;
#pragma unroll
    for (int e = 0; e < MAX_E; ++e) {
      const float w = e == e0 ? dl : (e == e1 ? -dl : 0.0f);
      acc[e][0] = fmaf(w, x.x, acc[e][0]);
      acc[e][1] = fmaf(w, x.y, acc[e][1]);
    }
  }
#pragma unroll
  for (int e = 0; e < MAX_E; ++e)
    if (e < E) {
      float* p = part + ((int64_t)blockIdx.x * E + e) * H + c;
      p[0] = acc[e][0];
      p[1] = acc[e][1];
    }
}

int grid_of(int64_t n, int per_block) {
  int64_t b = (n + per_block - 1) / per_block;
  if (b > 148 * 8) b = 148 * 8;
  return b < 1 ? 1 : (int)b;
}
}  // namespace

int moe_router_dw_blocks(int T) { return (T + RG_ROWS - 1) / RG_ROWS; }

void k_moe_router_fwd(const void* h2, const void* wr, float* g01, int T, int H, int E, cudaStream_t st) {
  moe_router_fwd_kernel<<<(T + WPB - 1) / WPB, WPB * 32, 0, st>>>((const bf16*)h2, (const bf16*)wr, g01, T, H, E);
  count_launch();
}
void k_moe_gather(const void* h2, void* X, int T, int H, int E, cudaStream_t st) {
  moe_gather_kernel<<<grid_of((int64_t)2 * T * H / 8, 256), 256, 0, st>>>((const bf16*)h2, (bf16*)X, T, H, E);
  count_launch();
}
void k_moe_combine(const void* x2, const void* O, const float* g01, void* y, int T, int H, int E, cudaStream_t st) {
  moe_combine_kernel<<<grid_of((int64_t)T * H / 8, 256), 256, 0, st>>>((const bf16*)x2, (const bf16*)O, g01, (bf16*)y,
                                                                        T, H, E);
  count_launch();
}
void k_moe_combine_bwd(const void* dy, const void* O, const float* g01, void* dO, float* dl0, int T, int H, int E,
                       cudaStream_t st) {
  moe_combine_bwd_kernel<<<(T + WPB - 1) / WPB, WPB * 32, 0, st>>>((const bf16*)dy, (const bf16*)O, g01, (bf16*)dO,
                                                                   dl0, T, H, E);
  count_launch();
}
void k_moe_router_bwd(const void* dX, const float* dl0, const void* wr, const void* h2, void* dh2, float* part,
                      int T, int H, int E, cudaStream_t st) {
  moe_router_dx_kernel<<<grid_of((int64_t)T * H / 8, 256), 256, 0, st>>>((const bf16*)dX, dl0, (const bf16*)wr,
                                                                          (bf16*)dh2, T, H, E);
  dim3 g(moe_router_dw_blocks(T), (H / 2 + 255) / 256);
  moe_router_dw_kernel<<<g, 256, 0, st>>>((const bf16*)h2, dl0, part, T, H, E);
  count_launch();
  count_launch();
}

cudaError_t preload_moe_kernels() {
  cudaFuncAttributes a;
  const void* fns[] = {(const void*)moe_router_fwd_kernel, (const void*)moe_gather_kernel,
                       (const void*)moe_combine_kernel, (const void*)moe_combine_bwd_kernel,
                       (const void*)moe_router_dx_kernel, (const void*)moe_router_dw_kernel};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace dc
