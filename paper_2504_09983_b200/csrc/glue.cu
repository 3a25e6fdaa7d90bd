// Glue kernels of the synthetic Llama-shaped layer and the
// counter-based parameter initialiser.  All HBM-bound, 16-byte vectorised,
// fp32 math, bf16 storage (RNE).  Row reductions use a fixed tree so results
// are deterministic run to run.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "act.cuh"
#include "dc_internal.h"

namespace dc {

using bf16 = __nv_bfloat16;
using bf162 = __nv_bfloat162;

// ------------------------------------------------------------------ generator
// value(seed, tensor_id, idx): splitmix64(seed ^ (tensor_id << 40) ^ idx),
// u = (h >> 40) * 2^-24, x = (u - 0.5f) * k.  Same recipe as synth/gen.py.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void init_param_kernel(uint64_t key, int64_t numel, int64_t base, int64_t S, float k,
                                  float* __restrict__ master, bf16* __restrict__ shard) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < S; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gi = base + j;
    float v = 0.0f;
    if (gi < numel) {
      if (k == 0.0f) {
        v = 1.0f;
      } else {
        const uint64_t h = splitmix64(key ^ (uint64_t)gi);
        const float u = __fmul_rn((float)(uint32_t)(h >> 40), 5.9604644775390625e-08f);  // 2^-24
        v = __fmul_rn(__fsub_rn(u, 0.5f), k);
      }
    }
    master[j] = v;
    shard[j] = __float2bfloat16_rn(v);
  }
}

void k_init_param(uint64_t seed, int32_t tensor_id, int64_t numel, int32_t world, int32_t rank, int64_t S,
                  float k, float* master, void* shard, cudaStream_t st) {
  const uint64_t key = seed ^ ((uint64_t)tensor_id << 40);
  int64_t blocks = (S + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  init_param_kernel<<<(int)blocks, 256, 0, st>>>(key, numel, (int64_t)rank * S, S, k, master,
                                                  reinterpret_cast<bf16*>(shard));
  count_launch();
}

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ void load8(const bf16* p, float (&f)[8]) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const bf162* h = reinterpret_cast<const bf162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ void store8(bf16* p, const float (&f)[8]) {
  uint4 u;
  bf162* h = reinterpret_cast<bf162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}

// block-wide sum, fixed order (warp shuffle tree, then warp 0 over warps)
template <int NT>
__device__ __forceinline__ float block_sum(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < NT / 32 ? sh[l] : 0.0f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0) sh[0] = v;
  }
  __syncthreads();
  float r = sh[0];
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------ RMSNorm
// h = bf16(x * rstd * g), rstd = 1/sqrt(mean(x^2) + eps).  One CTA per row.
constexpr int RN_T = 256;
__global__ void __launch_bounds__(RN_T) rmsnorm_fwd_kernel(const bf16* __restrict__ x, const bf16* __restrict__ g,
                                                          bf16* __restrict__ h, float* __restrict__ rstd, int H) {
  __shared__ float sh[32];
  const int64_t row = blockIdx.x;
  const bf16* xr = x + row * H;
  float ss = 0.0f;
  for (int c = threadIdx.x * 8; c < H; c += RN_T * 8) {
    float f[8];
    load8(xr + c, f);
#pragma unroll
    for (int i = 0; i < 8; ++i) ss = fmaf(f[i], f[i], ss);
  }
  ss = block_sum<RN_T>(ss, sh);
  const float r = 1.0f / sqrtf(ss / (float)H + 1e-5f);
  if (threadIdx.x == 0) rstd[row] = r;
  for (int c = threadIdx.x * 8; c < H; c += RN_T * 8) {
    float f[8], gg[8];
    load8(xr + c, f);
    load8(g + c, gg);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = f[i] * r * gg[i];
    store8(h + row * H + c, f);
  }
}

// Warp per row (default): no CTA-wide reduction, 8 rows per CTA in flight;
// the row is re-read from L1/L2 for the scaling pass.
__global__ void __launch_bounds__(256) rmsnorm_fwd_warp_kernel(const bf16* __restrict__ x, const bf16* __restrict__ g,
                                                              bf16* __restrict__ h, float* __restrict__ rstd, int T,
                                                              int H) {
  const int row = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= T) return;
  const bf16* xr = x + (int64_t)row * H;
  float ss = 0.0f;
  for (int c = lane * 8; c < H; c += 256) {
    float f[8];
    load8(xr + c, f);
#pragma unroll
    for (int i = 0; i < 8; ++i) ss = fmaf(f[i], f[i], ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float r = 1.0f / sqrtf(ss / (float)H + 1e-5f);
  if (lane == 0) rstd[row] = r;
  for (int c = lane * 8; c < H; c += 256) {
    float f[8], gg[8];
    load8(xr + c, f);
    load8(g + c, gg);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = f[i] * r * gg[i];
    store8(h + (int64_t)row * H + c, f);
  }
}

void k_rmsnorm_fwd(const void* x, const void* g, void* h, float* rstd, int T, int H, cudaStream_t st) {
  rmsnorm_fwd_warp_kernel<<<(T + 7) / 8, 256, 0, st>>>((const bf16*)x, (const bf16*)g, (bf16*)h, rstd, T, H);
  count_launch();
}

// dx = bf16(dres + rstd * (dn - n * mean(dn * n))), n = x*rstd, dn = dh*g;
// dg partial[blk][c] = sum over the block's rows of dh*n (fixed row order).
constexpr int RB_ROWS = 16;
int rmsnorm_bwd_blocks(int T) { return (T + RB_ROWS - 1) / RB_ROWS; }

// One pass per row: dh and x are loaded once into registers (CH chunks of 8
// columns per thread, H = CH * 2048), the gain once per CTA.
template <int CH>
__global__ void __launch_bounds__(RN_T) rmsnorm_bwd_kernel(const bf16* __restrict__ dh, const bf16* __restrict__ x,
                                                          const bf16* __restrict__ g, const float* __restrict__ rstd,
                                                          const bf16* __restrict__ dres, bf16* __restrict__ dx,
                                                          float* __restrict__ dgp, int T, int H) {
  __shared__ float sh[32];
  float acc[CH][8], gg[CH][8];
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c = threadIdx.x * 8 + j * RN_T * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[j][i] = 0.0f; gg[j][i] = 0.0f; }
    if (c < H) load8(g + c, gg[j]);
  }
  const int r0 = blockIdx.x * RB_ROWS;
  for (int rr = 0; rr < RB_ROWS; ++rr) {
    const int row = r0 + rr;
    if (row >= T) break;
    const float rs = rstd[row];
    const bf16* dhr = dh + (int64_t)row * H;
    const bf16* xr = x + (int64_t)row * H;
    float a[CH][8], n[CH][8], d[CH][8];
    float dot = 0.0f;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int c = threadIdx.x * 8 + j * RN_T * 8;
#pragma unroll
      for (int i = 0; i < 8; ++i) { a[j][i] = 0.0f; n[j][i] = 0.0f; d[j][i] = 0.0f; }
      if (c < H) {
        load8(dhr + c, a[j]);
        load8(xr + c, n[j]);
        if (dres) load8(dres + (int64_t)row * H + c, d[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < CH; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        n[j][i] = n[j][i] * rs;
        acc[j][i] += a[j][i] * n[j][i];
        dot = fmaf(a[j][i] * gg[j][i], n[j][i], dot);
      }
    dot = block_sum<RN_T>(dot, sh) / (float)H;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int c = threadIdx.x * 8 + j * RN_T * 8;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float base = dres ? d[j][i] : 0.0f;
        d[j][i] = base + rs * (a[j][i] * gg[j][i] - n[j][i] * dot);
      }
      if (c < H) store8(dx + (int64_t)row * H + c, d[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c = threadIdx.x * 8 + j * RN_T * 8;
    if (c < H) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dgp[(int64_t)blockIdx.x * H + c + i] = acc[j][i];
    }
  }
}

// Two-pass form (default): (1) one warp per row: dot[row] = sum_c dh g n
// (fixed lane order + shuffle tree); (2) a thread owns 8 columns of a 16-row
// chunk: dx = dres + rstd (dh g - n dot / H) and the dg partial of its columns,
// rows in order.  Every access is a coalesced 16-byte vector and nothing waits
// on a CTA-wide reduction, so the HBM pipe stays busy (the one-pass kernel
// above serialises a block reduction per row).
constexpr int RD_WARPS = 8;
__global__ void __launch_bounds__(RD_WARPS * 32) rmsnorm_bwd_dot_kernel(const bf16* __restrict__ dh,
                                                                      const bf16* __restrict__ x,
                                                                      const bf16* __restrict__ g,
                                                                      const float* __restrict__ rstd,
                                                                      float* __restrict__ dot, int T, int H) {
  const int row = blockIdx.x * RD_WARPS + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= T) return;
  const float rs = rstd[row];
  const bf16* dhr = dh + (int64_t)row * H;
  const bf16* xr = x + (int64_t)row * H;
  float s = 0.0f;
  for (int c = lane * 8; c < H; c += 256) {
    float a[8], n[8], gg[8];
    load8(dhr + c, a);
    load8(xr + c, n);
    load8(g + c, gg);
#pragma unroll
    for (int i = 0; i < 8; ++i) s = fmaf(a[i] * gg[i], n[i] * rs, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) dot[row] = s / (float)H;
}

__global__ void __launch_bounds__(256) rmsnorm_bwd_dx_kernel(const bf16* __restrict__ dh, const bf16* __restrict__ x,
                                                             const bf16* __restrict__ g,
                                                             const float* __restrict__ rstd,
                                                             const float* __restrict__ dot,
                                                             const bf16* __restrict__ dres, bf16* __restrict__ dx,
                                                             float* __restrict__ dgp, int T, int H) {
  const int c = (blockIdx.y * 256 + threadIdx.x) * 8;
  if (c >= H) return;
  float gg[8], acc[8];
  load8(g + c, gg);
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
  const int r0 = blockIdx.x * RB_ROWS;
  const int r1 = min(T, r0 + RB_ROWS);
#pragma unroll 4
  for (int row = r0; row < r1; ++row) {
    const float rs = rstd[row], dm = dot[row];
    float a[8], n[8], d[8];
    load8(dh + (int64_t)row * H + c, a);
    load8(x + (int64_t)row * H + c, n);
    if (dres) load8(dres + (int64_t)row * H + c, d);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      n[i] = n[i] * rs;
      acc[i] += a[i] * n[i];
      d[i] = (dres ? d[i] : 0.0f) + rs * (a[i] * gg[i] - n[i] * dm);
    }
    store8(dx + (int64_t)row * H + c, d);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) dgp[(int64_t)blockIdx.x * H + c + i] = acc[i];
}

// Single pass, warp per row (default for H = 256 NCH <= 4096): the row's dh
// and x stay in registers (bf16) between the dot and the dx pass, so each byte
// is read once; dg partials accumulate per warp in shared memory (each lane
// owns its columns: no atomics), then the 8 warps' rows are added in order.
template <int NCH>
__global__ void __launch_bounds__(256, 1) rmsnorm_bwd_row_kernel(const bf16* __restrict__ dh,
                                                                const bf16* __restrict__ x,
                                                                const bf16* __restrict__ g,
                                                                const float* __restrict__ rstd,
                                                                const bf16* __restrict__ dres, bf16* __restrict__ dx,
                                                                float* __restrict__ dgp, int T, int H) {
  extern __shared__ float wacc[];                      // [8 warps][H]
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  float* acc = wacc + (int64_t)w * H;
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    float4* a4 = reinterpret_cast<float4*>(acc + lane * 8 + k * 256);
    a4[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    a4[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int r0 = blockIdx.x * RB_ROWS, r1 = min(T, r0 + RB_ROWS);
  for (int row = r0 + w; row < r1; row += 8) {
    const bf16* dhr = dh + (int64_t)row * H;
    const bf16* xr = x + (int64_t)row * H;
    const float rs = rstd[row];
    float s = 0.0f;
#pragma unroll 4
    for (int k = 0; k < NCH; ++k) {        // pass 1: the row's dot (first read of dh, x)
      float a[8], n[8], gg[8];
      load8(dhr + lane * 8 + k * 256, a);
      load8(xr + lane * 8 + k * 256, n);
      load8(g + lane * 8 + k * 256, gg);
#pragma unroll
      for (int i = 0; i < 8; ++i) s = fmaf(a[i] * gg[i], n[i] * rs, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float dm = s / (float)H;
#pragma unroll 4
    for (int k = 0; k < NCH; ++k) {        // pass 2: dx and dg (the row is re-read from L1 / L2)
      const int c = lane * 8 + k * 256;
      float a[8], n[8], gg[8], d[8];
      load8(dhr + c, a);
      load8(xr + c, n);
      load8(g + c, gg);
      if (dres) load8(dres + (int64_t)row * H + c, d);
      float4* a4 = reinterpret_cast<float4*>(acc + c);     // 16-byte smem accesses: no bank conflicts
      float4 q0 = a4[0], q1 = a4[1];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        n[i] = n[i] * rs;
        d[i] = (dres ? d[i] : 0.0f) + rs * (a[i] * gg[i] - n[i] * dm);
      }
      q0.x += a[0] * n[0]; q0.y += a[1] * n[1]; q0.z += a[2] * n[2]; q0.w += a[3] * n[3];
      q1.x += a[4] * n[4]; q1.y += a[5] * n[5]; q1.z += a[6] * n[6]; q1.w += a[7] * n[7];
      a4[0] = q0;
      a4[1] = q1;
      store8(dx + (int64_t)row * H + c, d);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < H; c += 256) {
    float t = 0.0f;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += wacc[q * H + c];
    dgp[(int64_t)blockIdx.x * H + c] = t;
  }
}

void k_rmsnorm_bwd(const void* dh, const void* x, const void* g, const float* rstd, const void* dres, void* dx,
                   float* dg_partial, int T, int H, cudaStream_t st) {
  // default: two passes.  A/B (DC_RMSNORM_BWD): 1 one-pass CTA-per-rows kernel,
  // 3 warp-per-row single pass (measured 59.6 us vs 43.7 us for the two passes
  // at T = 4096, H = 4096: 128 KB of shared accumulators leave one CTA per SM)
  static const int form = getenv("DC_RMSNORM_BWD") ? atoi(getenv("DC_RMSNORM_BWD")) : 0;
  if (form == 3 && H % 256 == 0 && H <= 4096) {
    const size_t smem = (size_t)8 * H * 4;
#define DC_RR(NCH_)                                                                                \
    rmsnorm_bwd_row_kernel<NCH_><<<rmsnorm_bwd_blocks(T), 256, smem, st>>>(                         \
        (const bf16*)dh, (const bf16*)x, (const bf16*)g, rstd, (const bf16*)dres, (bf16*)dx, dg_partial, T, H)
    switch (H / 256) {
      case 1: DC_RR(1); break;
      case 2: DC_RR(2); break;
      case 4: DC_RR(4); break;
      case 8: DC_RR(8); break;
      case 16: DC_RR(16); break;
      default: goto two_pass;
    }
#undef DC_RR
    count_launch();
    return;
  }
two_pass:
  if (form != 1) {
    float* dot = dg_partial + (int64_t)rmsnorm_bwd_blocks(T) * H;    // T floats of scratch after the partials
    rmsnorm_bwd_dot_kernel<<<(T + RD_WARPS - 1) / RD_WARPS, RD_WARPS * 32, 0, st>>>(
        (const bf16*)dh, (const bf16*)x, (const bf16*)g, rstd, dot, T, H);
    dim3 grid(rmsnorm_bwd_blocks(T), (H / 8 + 255) / 256);
    rmsnorm_bwd_dx_kernel<<<grid, 256, 0, st>>>((const bf16*)dh, (const bf16*)x, (const bf16*)g, rstd, dot,
                                                 (const bf16*)dres, (bf16*)dx, dg_partial, T, H);
    count_launch();
    count_launch();
    return;
  }
  const int ch = (H + RN_T * 8 - 1) / (RN_T * 8);
#define DC_RB(CH_)                                                                                  \
  rmsnorm_bwd_kernel<CH_><<<rmsnorm_bwd_blocks(T), RN_T, 0, st>>>((const bf16*)dh, (const bf16*)x,     \
      (const bf16*)g, rstd, (const bf16*)dres, (bf16*)dx, dg_partial, T, H)
  if (ch == 1) DC_RB(1);
  else if (ch == 2) DC_RB(2);
  else if (ch == 3) DC_RB(3);
  else DC_RB(4);
#undef DC_RB
  count_launch();
}

// One pass (default): a CTA of up to 512 threads owns the whole width (each
// thread 8 x CH columns) and a contiguous range of rows, processed in groups
// of RBF rows.  Per group every input byte is read once: dh and x (prefetched
// one group ahead, so their loads are in flight during the previous group's
// reduction), the group's RBF row dots are reduced together (one CTA barrier
// per group instead of per row), then dx = dres + rstd (dh g - n dot / H) is
// written and the thread's dg columns accumulate (rows in order).  The last
// CTA to finish (counter) adds the per-CTA dg partials in CTA order and
// writes bf16 dg, so no separate column-sum launch.  Deterministic.
constexpr int RBF = 4;
template <int CH>
__global__ void __launch_bounds__(512, 1) rmsnorm_bwd_fused_kernel(
    const bf16* __restrict__ dh, const bf16* __restrict__ x, const bf16* __restrict__ g,
    const float* __restrict__ rstd, const bf16* __restrict__ dres, bf16* __restrict__ dx, float* __restrict__ part,
    uint32_t* __restrict__ counter, bf16* __restrict__ dg, int T, int H, int rows_per_cta) {
  __shared__ float red[2][RBF][16];
  __shared__ int last;
  const int nt = blockDim.x, nw = nt / 32, w = threadIdx.x / 32, lane = threadIdx.x % 32;
  float gg[CH][8], acc[CH][8];
  bool ok[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c = (threadIdx.x + j * nt) * 8;
    ok[j] = c < H;
#pragma unroll
    for (int i = 0; i < 8; ++i) { gg[j][i] = 0.0f; acc[j][i] = 0.0f; }
    if (ok[j]) load8(g + c, gg[j]);
  }
  const int r0 = blockIdx.x * rows_per_cta, r1 = min(T, r0 + rows_per_cta);
  uint4 A[RBF][CH], X[RBF][CH];
  auto fetch = [&](int rb) {
#pragma unroll
    for (int r = 0; r < RBF; ++r)
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = (threadIdx.x + j * nt) * 8;
        if (rb + r < r1 && ok[j]) {
          A[r][j] = *reinterpret_cast<const uint4*>(dh + (int64_t)(rb + r) * H + c);
          X[r][j] = *reinterpret_cast<const uint4*>(x + (int64_t)(rb + r) * H + c);
        }
      }
  };
  if (r0 < r1) fetch(r0);
  int buf = 0;
  for (int rb = r0; rb < r1; rb += RBF, buf ^= 1) {
    float a[RBF][CH][8], n[RBF][CH][8], rs[RBF], sdot[RBF];
#pragma unroll
    for (int r = 0; r < RBF; ++r) {
      rs[r] = rb + r < r1 ? rstd[rb + r] : 0.0f;
      sdot[r] = 0.0f;
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const bf162* ha = reinterpret_cast<const bf162*>(&A[r][j]);
        const bf162* hx = reinterpret_cast<const bf162*>(&X[r][j]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 fa = __bfloat1622float2(ha[i]), fx = __bfloat1622float2(hx[i]);
          a[r][j][2 * i] = fa.x; a[r][j][2 * i + 1] = fa.y;
          n[r][j][2 * i] = fx.x * rs[r]; n[r][j][2 * i + 1] = fx.y * rs[r];
        }
        if (!(rb + r < r1 && ok[j]))
#pragma unroll
          for (int i = 0; i < 8; ++i) { a[r][j][i] = 0.0f; n[r][j][i] = 0.0f; }
#pragma unroll
        for (int i = 0; i < 8; ++i) sdot[r] = fmaf(a[r][j][i] * gg[j][i], n[r][j][i], sdot[r]);
      }
    }
    if (rb + RBF < r1) fetch(rb + RBF);      // next group's loads in flight across the reduction
#pragma unroll
    for (int r = 0; r < RBF; ++r) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sdot[r] += __shfl_xor_sync(0xffffffffu, sdot[r], o);
      if (lane == 0) red[buf][r][w] = sdot[r];
    }
    __syncthreads();                          // (double-buffered `red`: one barrier per group)
#pragma unroll
    for (int r = 0; r < RBF; ++r) {
      float t = 0.0f;
      for (int q = 0; q < nw; ++q) t += red[buf][r][q];   // warp order: fixed
      sdot[r] = t / (float)H;
    }
#pragma unroll
    for (int r = 0; r < RBF; ++r) {
      if (rb + r >= r1) continue;
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        if (!ok[j]) continue;
        const int c = (threadIdx.x + j * nt) * 8;
        float d[8];
        if (dres) load8(dres + (int64_t)(rb + r) * H + c, d);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          acc[j][i] += a[r][j][i] * n[r][j][i];
          d[i] = (dres ? d[i] : 0.0f) + rs[r] * (a[r][j][i] * gg[j][i] - n[r][j][i] * sdot[r]);
        }
        store8(dx + (int64_t)(rb + r) * H + c, d);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c = (threadIdx.x + j * nt) * 8;
    if (ok[j]) {
      float4* p4 = reinterpret_cast<float4*>(part + (int64_t)blockIdx.x * H + c);
      p4[0] = make_float4(acc[j][0], acc[j][1], acc[j][2], acc[j][3]);
      p4[1] = make_float4(acc[j][4], acc[j][5], acc[j][6], acc[j][7]);
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int c = threadIdx.x; c < H; c += nt) {       // CTA order: deterministic
    float t = 0.0f;
    for (int b = 0; b < (int)gridDim.x; ++b) t += __ldcg(part + (int64_t)b * H + c);
    dg[c] = __float2bfloat16_rn(t);
  }
  if (threadIdx.x == 0) *counter = 0u;               // ready for the next launch
}

int rmsnorm_bwd_fused_grid(int T) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1) sms = 148;
  }
  const int g = (T + RBF - 1) / RBF;
  return g < sms ? g : sms;
}

dc_status k_rmsnorm_bwd_dg(const void* dh, const void* x, const void* g, const float* rstd, const void* dres, void* dx,
                           void* dg, float* part, uint32_t* counter, int T, int H, cudaStream_t st) {
  if (H % 8 || H > 8192) return DC_EINVAL;
  const int grid = rmsnorm_bwd_fused_grid(T);
  const int rows = (T + grid - 1) / grid;
  int nt = H / 8 < 512 ? H / 8 : 512;
  nt = (nt + 31) / 32 * 32;
  if (H <= 8 * nt)
    rmsnorm_bwd_fused_kernel<1><<<grid, nt, 0, st>>>((const bf16*)dh, (const bf16*)x, (const bf16*)g, rstd,
                                                     (const bf16*)dres, (bf16*)dx, part, counter, (bf16*)dg, T, H, rows);
  else
    rmsnorm_bwd_fused_kernel<2><<<grid, nt, 0, st>>>((const bf16*)dh, (const bf16*)x, (const bf16*)g, rstd,
                                                     (const bf16*)dres, (bf16*)dx, part, counter, (bf16*)dg, T, H, rows);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? DC_OK : DC_ECUDA;
}

// out[c] = bf16(sum_b p[b][c]): a CTA owns 32 columns; warp w sums rows
// w, w + 8, ... (coalesced 128 B per row), then the 8 partials are added in
// warp order (fixed, deterministic)
__global__ void __launch_bounds__(256) colsum_kernel(const float* __restrict__ p, int nblk, int H,
                                                     bf16* __restrict__ out) {
  __shared__ float sh[8][33];
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  const int c = blockIdx.x * 32 + lane;
  float s = 0.0f;
  if (c < H)
    for (int b = w; b < nblk; b += 8) s += p[(int64_t)b * H + c];
  sh[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < H) {
    float t = 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sh[k][lane];
    out[c] = __float2bfloat16_rn(t);
  }
}

void k_colsum_to_bf16(const float* partial, int nblk, int H, void* out, cudaStream_t st) {
  colsum_kernel<<<(H + 31) / 32, 256, 0, st>>>(partial, nblk, H, (bf16*)out);
  count_launch();
}

// ------------------------------------------------------------------ attention surrogate
// a = bf16(q + rep(k) * rep(v)); qkv row = [q (qd) | k (kvd) | v (kvd)].
__global__ void attn_mix_fwd_kernel(const bf16* __restrict__ qkv, bf16* __restrict__ a, int T, int qd, int kvd,
                                    int hd, int grp) {
  const int ld = qd + 2 * kvd;
  const int64_t n8 = (int64_t)T * qd / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 8;
    const int t = (int)(e / qd), c = (int)(e % qd);
    const int head = c / hd, d = c % hd;
    const int kc = (head / grp) * hd + d;
    const bf16* row = qkv + (int64_t)t * ld;
    float q[8], k[8], v[8], o[8];
    load8(row + c, q);
    load8(row + qd + kc, k);
    load8(row + qd + kvd + kc, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = fmaf(k[j], v[j], q[j]);
    store8(a + e, o);
  }
}

static int grid_for(int64_t n, int per_block) {
  int64_t b = (n + per_block - 1) / per_block;
  if (b > 148 * 8) b = 148 * 8;
  return b < 1 ? 1 : (int)b;
}

void k_attn_mix_fwd(const void* qkv, void* a, int T, int qd, int kvd, int hd, int grp, cudaStream_t st) {
  attn_mix_fwd_kernel<<<grid_for((int64_t)T * qd / 8, 256), 256, 0, st>>>((const bf16*)qkv, (bf16*)a, T, qd, kvd,
                                                                           hd, grp);
  count_launch();
}

// dqkv row = [dq = da (already written by the o-projection dX GEMM) | dk | dv]
// dk[j*hd+d] = sum_{h in group j} da[h*hd+d] * v[j*hd+d]; dv likewise with k.
__global__ void attn_mix_bwd_kernel(bf16* __restrict__ dqkv, const bf16* __restrict__ qkv, int T, int qd, int kvd,
                                    int hd, int grp) {
  const int ld = qd + 2 * kvd;
  const int64_t n8 = (int64_t)T * kvd / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 8;
    const int t = (int)(e / kvd), kc = (int)(e % kvd);
    const int j = kc / hd, d = kc % hd;
    const bf16* row = qkv + (int64_t)t * ld;
    bf16* drow = dqkv + (int64_t)t * ld;
    float k[8], v[8], sk[8], sv[8];
    load8(row + qd + kc, k);
    load8(row + qd + kvd + kc, v);
#pragma unroll
    for (int x = 0; x < 8; ++x) { sk[x] = 0.0f; sv[x] = 0.0f; }
    for (int h = j * grp; h < (j + 1) * grp; ++h) {
      float da[8];
      load8(drow + h * hd + d, da);
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        sk[x] = fmaf(da[x], v[x], sk[x]);
        sv[x] = fmaf(da[x], k[x], sv[x]);
      }
    }
    store8(drow + qd + kc, sk);
    store8(drow + qd + kvd + kc, sv);
  }
}

void k_attn_mix_bwd(void* dqkv, const void* qkv, int T, int qd, int kvd, int hd, int grp, cudaStream_t st) {
  attn_mix_bwd_kernel<<<grid_for((int64_t)T * kvd / 8, 256), 256, 0, st>>>((bf16*)dqkv, (const bf16*)qkv, T, qd,
                                                                            kvd, hd, grp);
  count_launch();
}

// ------------------------------------------------------------------ SiLU * up
__global__ void act_fwd_kernel(const bf16* __restrict__ gu, bf16* __restrict__ act, int T, int F) {
  const int64_t n8 = (int64_t)T * F / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 8;
    const int t = (int)(e / F), c = (int)(e % F);
    const bf16* row = gu + (int64_t)t * 2 * F;
    float g[8], u[8], o[8];
    load8(row + c, g);
    load8(row + F + c, u);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = silu_mul(g[j], u[j]);
    store8(act + e, o);
  }
}

void k_act_fwd(const void* gu, void* act, int T, int F, cudaStream_t st) {
  act_fwd_kernel<<<grid_for((int64_t)T * F / 8, 256), 256, 0, st>>>((const bf16*)gu, (bf16*)act, T, F);
  count_launch();
}

// d_gate = bf16(dact * up * silu'(g)), d_up = bf16(dact * silu(g))
__global__ void act_bwd_kernel(const bf16* __restrict__ dact, const bf16* __restrict__ gu, bf16* __restrict__ dgu,
                               int T, int F) {
  const int64_t n8 = (int64_t)T * F / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 8;
    const int t = (int)(e / F), c = (int)(e % F);
    const bf16* row = gu + (int64_t)t * 2 * F;
    float g[8], u[8], da[8], dg[8], du[8];
    load8(row + c, g);
    load8(row + F + c, u);
    load8(dact + e, da);
#pragma unroll
    for (int j = 0; j < 8; ++j) silu_mul_bwd(da[j], g[j], u[j], dg[j], du[j]);
    store8(dgu + (int64_t)t * 2 * F + c, dg);
    store8(dgu + (int64_t)t * 2 * F + F + c, du);
  }
}

void k_act_bwd(const void* dact, const void* gu, void* dgu, int T, int F, cudaStream_t st) {
  act_bwd_kernel<<<grid_for((int64_t)T * F / 8, 256), 256, 0, st>>>((const bf16*)dact, (const bf16*)gu, (bf16*)dgu,
                                                                     T, F);
  count_launch();
}

// ------------------------------------------------------------------ loss
// loss = mean 1/2 (y - t)^2 ; dy = bf16((y - t) / n).  Deterministic 2-pass sum.
constexpr int LOSS_BLOCKS = 296;
__global__ void loss_kernel(const bf16* __restrict__ y, const bf16* __restrict__ t, bf16* __restrict__ dy,
                            float* __restrict__ partial, int64_t n) {
  __shared__ float sh[32];
  const float inv = 1.0f / (float)n;
  float s = 0.0f;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 8; i < n; i += (int64_t)gridDim.x * blockDim.x * 8) {
    float a[8], b[8], d[8];
    load8(y + i, a);
    load8(t + i, b);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float e = a[j] - b[j];
      s = fmaf(0.5f * e, e, s);
      d[j] = e * inv;
    }
    store8(dy + i, d);
  }
  s = block_sum<256>(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}
__global__ void loss_final_kernel(const float* __restrict__ partial, int nb, int64_t n, float* __restrict__ loss) {
  __shared__ float sh[32];
  float s = 0.0f;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += partial[i];
  s = block_sum<256>(s, sh);
  if (threadIdx.x == 0) *loss = (float)((double)s / (double)n);
}

void k_loss(const void* y, const void* t, void* dy, float* partial, float* loss, int64_t n, cudaStream_t st) {
  loss_kernel<<<LOSS_BLOCKS, 256, 0, st>>>((const bf16*)y, (const bf16*)t, (bf16*)dy, partial, n);
  loss_final_kernel<<<1, 256, 0, st>>>(partial, LOSS_BLOCKS, n, loss);
  count_launch();
  count_launch();
}

void k_zero(void* p, int64_t bytes, cudaStream_t st) {
  cudaMemsetAsync(p, 0, bytes, st);
}

}  // namespace dc

namespace dc {
cudaError_t preload_glue_kernels() {
  cudaFuncAttributes a;
  const void* fns[] = {(const void*)init_param_kernel, (const void*)rmsnorm_fwd_kernel,
                       (const void*)rmsnorm_bwd_kernel<1>, (const void*)rmsnorm_bwd_kernel<2>,
                       (const void*)rmsnorm_bwd_kernel<3>, (const void*)rmsnorm_bwd_kernel<4>, (const void*)colsum_kernel,
                       (const void*)rmsnorm_bwd_dot_kernel, (const void*)rmsnorm_bwd_dx_kernel,
                       (const void*)rmsnorm_fwd_warp_kernel,
                       (const void*)rmsnorm_bwd_fused_kernel<1>, (const void*)rmsnorm_bwd_fused_kernel<2>,
                       (const void*)rmsnorm_bwd_row_kernel<1>, (const void*)rmsnorm_bwd_row_kernel<2>,
                       (const void*)rmsnorm_bwd_row_kernel<4>, (const void*)rmsnorm_bwd_row_kernel<8>,
                       (const void*)rmsnorm_bwd_row_kernel<16>,
                       (const void*)attn_mix_fwd_kernel, (const void*)attn_mix_bwd_kernel,
                       (const void*)act_fwd_kernel, (const void*)act_bwd_kernel,
                       (const void*)loss_kernel, (const void*)loss_final_kernel};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  const void* rows[] = {(const void*)rmsnorm_bwd_row_kernel<1>, (const void*)rmsnorm_bwd_row_kernel<2>,
                        (const void*)rmsnorm_bwd_row_kernel<4>, (const void*)rmsnorm_bwd_row_kernel<8>,
                        (const void*)rmsnorm_bwd_row_kernel<16>};
  const int nch[] = {1, 2, 4, 8, 16};
  for (int i = 0; i < 5; ++i) {
    cudaError_t e = cudaFuncSetAttribute(rows[i], cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * nch[i] * 256 * 4);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}
}  // namespace dc
