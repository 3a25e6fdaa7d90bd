// bf16 GEMM on the 5th-generation tensor cores (sm_100a):
//   C[M,N] (bf16) = A_op[M,K] * B_op[K,N] (+ R)   with fp32 accumulation in TMEM.
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      TMA producer (one elected lane): A/B tiles -> 4-stage smem ring
//   warp 1      MMA issuer (one lane): tcgen05.mma 128x256x16, accumulators in
//               TMEM (2 x 256 columns, double buffered across tiles)
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: tcgen05.ld -> registers -> (+R) -> bf16 -> global
// Operand majorness per operand (K-major, or MN-major through the UMMA
// descriptor's transpose bit), so the three layer GEMMs need no transposes:
//   forward  Y  = X  W^T : A K-major,  B K-major
//   backward dX = dY W   : A K-major,  B MN-major
//   backward dW = dY^T X : A MN-major, B MN-major
// B may be split into up to 4 segments along N (fused q|k|v and gate|up
// projections read three / two gathered tensors) or along K (their dX).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>

#include "act.cuh"
#include "adam.cuh"
#include "dc_internal.h"
#include "ptx.cuh"

namespace dc {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4, UMMA_K = 16;
constexpr int A_STAGE = BM * BK * 2;          // 16 KiB
constexpr int B_STAGE = BN * BK * 2;          // 32 KiB
constexpr int GEMM_THREADS = 256;
constexpr int TMEM_COLS = 512;
constexpr int GEMM_SMEM = STAGES * (A_STAGE + B_STAGE) + 1024 /*align*/ + 256 /*barriers*/;

struct GemmParams {
  int M, N, K;
  int m_tiles, n_tiles, k_blocks;
  int nseg, split_k;
  int seg_end[4];      // cumulative, in n-tiles (split N) or k-blocks (split K)
  int a_mn, b_mn;
  __nv_bfloat16* C;
  int64_t ldc;
  const __nv_bfloat16* R;
  int64_t ldr;
  uint32_t idesc;
  // epilogue mode 1 (fused reduce-scatter + Adam at N = 1): C[row, col] is the
  // gradient of element row * ldc + col of a parameter whose fp32 master/m/v
  // and bf16 shard are given; Adam scalars as in rs_adam (reading D18)
  int epi;
  float* master;
  float* m;
  float* v;
  __nv_bfloat16* shard;
  float w1, w2, b2, neg_s, c, eps;
  // side job (pair kernel, N = 1): groups [g0, g1) of 8 shard elements of a
  // previous layer's reduce-scatter + Adam, streamed by 6 otherwise idle warps
  // while the tensor cores run this GEMM (same arithmetic as rs_adam)
  SideJob side;
  // epilogue modes 2 / 3 (pair kernel): SiLU(gate) * up fused into the gate|up
  // GEMM (2: C = gu gate half, C + glu_off = up half, aux = act) and its
  // backward into the down-projection dX GEMM (3: acc = dact, aux = gu,
  // C = d(gate), C + glu_off = d(up)); N = F there
  __nv_bfloat16* aux;
  int64_t ld_aux, glu_off;
  int group_m;         // tile order: m-tiles per group (tile_mn)
  // stream-K tail (pair kernel): tiles [0, sk_dp) are data-parallel (tile t on
  // pair t % npairs); the remaining tiles' k-blocks [0, sk_total) are split into
  // npairs contiguous ranges.  A tile cut by a range boundary is computed in two
  // parts: the head's fp32 partial goes through sk_ws (flag sk_flags = sk_epoch),
  // the pair holding the tail adds it in its epilogue, which it runs last.
  // half-width tail (pair kernel, plain epilogue, no stream-K): tiles [0, ht_dp)
  // run whole; each remaining tile of the partial last wave runs as two
  // 256 x 128 halves (UMMA N = 128, instruction descriptor idesc_half), so that
  // wave has twice as many, half-length units for the idle pairs
  int ht_on, ht_dp;
  uint32_t idesc_half;
  int sk_on, sk_dp;
  int64_t sk_total;
  float* sk_ws;
  uint32_t* sk_flags;
  uint32_t sk_epoch;
  // fused all-gather -> GEMM (dc_gemm_args.chunk_*): per B segment
  const uint32_t* cf[4];
  int64_t cS[4], cE[4], cn[4], cld[4];
  uint32_t cval[4];
  uint32_t* cerr;
  uint64_t ctmo;
};

__device__ __forceinline__ uint32_t ld_acquire_cta(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(ptx::smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" :: "r"(ptx::smem_u32(p)), "r"(v) : "memory");
}

// Wait until every gather chunk overlapping flat elements [e0, e1) of B
// segment s has landed (fused all-gather -> GEMM), called by a whole warp (the
// watcher; warp-uniform arguments).  Chunks in linear order L = q nj + j
// (sender q, j-th of nj = ceil(S / E) chunks; word flags[q * 64 + j]): the 32
// lanes test chunks L .. L + 31 with one acquire load each, so a run of chunks
// that already landed costs one round trip, not one per chunk; the first chunk
// not landed yet is then awaited.  Keeps going past e1 over chunks that
// already landed (up to 32 at a time) and returns the flat end of the last
// verified chunk — the caller's cache.  Scalars by value: a reference to the
// kernel's GemmParams would put the whole parameter block in local memory.
__device__ __noinline__ int64_t chunk_wait(const uint32_t* flags, int64_t S, int64_t E, int64_t numel, uint32_t value,
                                           uint32_t* err, uint64_t tmo, int64_t e0, int64_t e1) {
  const int lane = threadIdx.x % 32;
  e1 = e1 < numel ? e1 : numel;
  if (e0 >= e1) return e1;
  const int64_t nj = (S + E - 1) / E;
  const int64_t nL = ((numel + S - 1) / S) * nj;     // chunks that exist
  auto chunk_end = [&](int64_t L) {                  // flat end of linear chunk L
    const int64_t q = L / nj, j = L - q * nj;
    return q * S + ((j + 1) * E < S ? (j + 1) * E : S);
  };
  int64_t L = (e0 / S) * nj + (e0 - (e0 / S) * S) / E;
  uint64_t t0 = 0;
  while (true) {
    const int64_t Ll = L + lane;
    bool ok = true;
    uint32_t seen = value;
    if (Ll < nL) {
      seen = ptx::ld_acquire_sys(flags + (Ll / nj) * AG_CHUNKS + (Ll % nj));
      ok = (int32_t)(seen - value) >= 0;
    }
    const uint32_t bad = __ballot_sync(0xffffffffu, !ok);
    const int f = bad ? __ffs(bad) - 1 : 32;          // chunks L .. L + f - 1 landed
    if (f > 0) {
      L += f;
      t0 = 0;
      if (L >= nL || chunk_end(L - 1) >= e1) {         // the range is covered
        if (bad || L >= nL) return chunk_end(L - 1);
        continue;                                      // all 32 landed: look further ahead
      }
      continue;
    }
    // chunk L itself has not landed: wait (bounded), fail fast after any timeout
    if (!t0) t0 = ptx::globaltimer();
    if ((err && *reinterpret_cast<volatile uint32_t*>(err)) || ptx::globaltimer() - t0 > tmo) {
      if (lane == 0 && err && !*reinterpret_cast<volatile uint32_t*>(err) && atomicCAS(err + 1, 0u, 1u) == 0u) {
        const uint32_t* fp = flags + (L / nj) * AG_CHUNKS + (L % nj);
        err[2] = value;
        err[3] = __shfl_sync(0x1u, seen, 0);
        err[4] = (uint32_t)reinterpret_cast<uintptr_t>(fp);
        err[5] = (uint32_t)(reinterpret_cast<uintptr_t>(fp) >> 32);
        __threadfence_system();
        atomicExch(err, 0x600u);
      }
      __syncwarp();
      return e1;
    }
    __nanosleep(128);
  }
}
// Tile order (tile index -> (m-tile, n-tile)): m fastest inside groups of
// group_m m-tiles (group_m = m_tiles: m fastest over all of them).  When
// m_tiles >> n_tiles (the gate / up dW GEMMs: 56 x 16 tiles) small groups make
// the resident CTA pairs sweep every n-column of a few m-rows: B stays in L2
// and A is streamed once, instead of all of A once per wave (launch_gemm).
#ifndef DC_GEMM_GROUP_DEFAULT
#define DC_GEMM_GROUP_DEFAULT 2
#endif
__device__ __forceinline__ void tile_mn(const GemmParams& p, int tile, int& mt, int& nt) {
  const int per = p.group_m * p.n_tiles;
  const int g = tile / per, r = tile - g * per;
  const int mb = g * p.group_m;
  const int gm = min(p.group_m, p.m_tiles - mb);
  mt = mb + r % gm;
  nt = r / gm;
}


// One unit of a pair's work list: k-blocks [kb0, kb1) of `tile`;
// mode 0 full tile, 1 head of a split tile (write fp32 partial), 2 tail (add it)
struct Unit { int tile, kb0, kb1, mode, half; };   // half: -1 whole tile, 0 / 1 the 128-column halves

struct WorkList {
  int n_dp, n_rest, finish;     // DP tiles, SK units (or half-tail units) without a wait, trailing tail unit
  int ta, ka, tb;               // first SK tile / its start k-block, first non-tail SK tile
  int64_t s1;                   // end of this pair's SK range (k-block index)
  __device__ __forceinline__ int count() const { return n_dp + n_rest + finish; }
};

template <bool HT = false>
__device__ __forceinline__ WorkList work_list(const GemmParams& p, int pair, int npairs) {
  WorkList w{};
  const int tiles = p.m_tiles * p.n_tiles;
  const int dp = p.sk_on ? p.sk_dp : (HT && p.ht_on) ? p.ht_dp : tiles;
  w.n_dp = pair < dp ? (dp - 1 - pair) / npairs + 1 : 0;
  if constexpr (HT) {
    if (p.ht_on) {                               // half units h = pair, pair + npairs, ... < 2 (tiles - dp)
      const int nh = 2 * (tiles - dp);
      w.n_rest = pair < nh ? (nh - 1 - pair) / npairs + 1 : 0;
      return w;
    }
  }
  if (!p.sk_on) return w;
  const int KB = p.k_blocks;
  const int64_t s0 = (int64_t)pair * p.sk_total / npairs;
  w.s1 = (int64_t)(pair + 1) * p.sk_total / npairs;
  w.ta = dp + (int)(s0 / KB);
  w.ka = (int)(s0 % KB);
  w.finish = w.ka != 0;                         // ranges are >= KB long: the tail ends its tile
  w.tb = w.ta + w.finish;
  const int64_t first = (int64_t)(w.tb - dp) * KB;
  w.n_rest = w.s1 > first ? (int)((w.s1 - first + KB - 1) / KB) : 0;
  return w;
}

template <bool HT = false>
__device__ __forceinline__ Unit unit_at(const GemmParams& p, const WorkList& w, int pair, int npairs, int i) {
  Unit u;
  u.half = -1;
  if (i < w.n_dp) { u.tile = pair + i * npairs; u.kb0 = 0; u.kb1 = p.k_blocks; u.mode = 0; return u; }
  i -= w.n_dp;
  if constexpr (HT) {
    if (p.ht_on) {
      const int h = pair + i * npairs;
      u.tile = p.ht_dp + h / 2; u.half = h % 2; u.kb0 = 0; u.kb1 = p.k_blocks; u.mode = 0;
      return u;
    }
  }
  const int KB = p.k_blocks;
  if (i < w.n_rest) {
    u.tile = w.tb + i;
    u.kb0 = 0;
    const int64_t end = w.s1 - (int64_t)(u.tile - p.sk_dp) * KB;
    u.kb1 = end < KB ? (int)end : KB;
    u.mode = u.kb1 < KB ? 1 : 0;
    return u;
  }
  u.tile = w.ta; u.kb0 = w.ka; u.kb1 = KB; u.mode = 2;
  return u;
}

__device__ __forceinline__ int seg_of(const GemmParams& p, int idx) {
  int s = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
    if (i + 1 < p.nseg && idx >= p.seg_end[i]) s = i + 1;
  return s;
}


// One 32-column chunk of an accumulator row (thread = row) -> global memory.
// Mode 0: C = bf16(acc [+ R]).  Mode 1 (N = 1 fused reduce-scatter + Adam):
// g = fp32(bf16(acc)) is exactly the value the grad slot would hold, x 1/N
// (= 1), then the fp32 Adam step of rs_adam on master/m/v (same op order,
// same intrinsics, no FMA) and the bf16 shard; nothing is written to C.
template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int row, int col0, const uint32_t (&v)[32]) {
  float f[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
  const bool full = col0 + 32 <= p.N;
  if constexpr (EPI == 1) {
    const int64_t e0 = (int64_t)row * p.ldc + col0;
    if (full) {
      float4 P[8], Mv[8], V[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        P[t] = reinterpret_cast<const float4*>(p.master + e0)[t];
        Mv[t] = reinterpret_cast<const float4*>(p.m + e0)[t];
        V[t] = reinterpret_cast<const float4*>(p.v + e0)[t];
      }
      uint4 sh[4];
      __nv_bfloat162* s2 = reinterpret_cast<__nv_bfloat162*>(sh);
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        float pp[4] = {P[t].x, P[t].y, P[t].z, P[t].w};
        float mm[4] = {Mv[t].x, Mv[t].y, Mv[t].z, Mv[t].w};
        float vv[4] = {V[t].x, V[t].y, V[t].z, V[t].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float g = __bfloat162float(__float2bfloat16_rn(f[4 * t + u]));
          const float mj = __fadd_rn(mm[u], __fmul_rn(p.w1, __fsub_rn(g, mm[u])));
          const float vj = __fadd_rn(__fmul_rn(p.b2, vv[u]), __fmul_rn(__fmul_rn(p.w2, g), g));
          const float d = __fadd_rn(__fdiv_rn(__fsqrt_rn(vj), p.c), p.eps);
          pp[u] = __fadd_rn(pp[u], __fdiv_rn(__fmul_rn(p.neg_s, mj), d));
          mm[u] = mj;
          vv[u] = vj;
        }
        reinterpret_cast<float4*>(p.master + e0)[t] = make_float4(pp[0], pp[1], pp[2], pp[3]);
        reinterpret_cast<float4*>(p.m + e0)[t] = make_float4(mm[0], mm[1], mm[2], mm[3]);
        reinterpret_cast<float4*>(p.v + e0)[t] = make_float4(vv[0], vv[1], vv[2], vv[3]);
        s2[2 * t] = __floats2bfloat162_rn(pp[0], pp[1]);
        s2[2 * t + 1] = __floats2bfloat162_rn(pp[2], pp[3]);
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) reinterpret_cast<uint4*>(p.shard + e0)[t] = sh[t];
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (col0 + j >= p.N) continue;
        const int64_t e = e0 + j;
        const float g = __bfloat162float(__float2bfloat16_rn(f[j]));
        const float mj = __fadd_rn(p.m[e], __fmul_rn(p.w1, __fsub_rn(g, p.m[e])));
        const float vj = __fadd_rn(__fmul_rn(p.b2, p.v[e]), __fmul_rn(__fmul_rn(p.w2, g), g));
        const float d = __fadd_rn(__fdiv_rn(__fsqrt_rn(vj), p.c), p.eps);
        const float pj = __fadd_rn(p.master[e], __fdiv_rn(__fmul_rn(p.neg_s, mj), d));
        p.master[e] = pj; p.m[e] = mj; p.v[e] = vj;
        p.shard[e] = __float2bfloat16_rn(pj);
      }
    }
    return;
  }
  __nv_bfloat16* crow = p.C + (int64_t)row * p.ldc;
  if (p.R) {
    const __nv_bfloat16* rrow = p.R + (int64_t)row * p.ldr;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 rv = *reinterpret_cast<const uint4*>(rrow + col0 + j);
        const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&rv);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          float2 rf = __bfloat1622float2(r2[t]);
          f[j + 2 * t] = __fadd_rn(f[j + 2 * t], rf.x);
          f[j + 2 * t + 1] = __fadd_rn(f[j + 2 * t + 1], rf.y);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < p.N) f[j] = __fadd_rn(f[j], __bfloat162float(rrow[col0 + j]));
    }
  }
  if (full) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint4 o;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int t = 0; t < 4; ++t) o2[t] = __floats2bfloat162_rn(f[j + 2 * t], f[j + 2 * t + 1]);
      *reinterpret_cast<uint4*>(crow + col0 + j) = o;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j < p.N) crow[col0 + j] = __float2bfloat16_rn(f[j]);
  }
}

// GLU forward (mode 2), one 32-column chunk of a row: gate / up accumulators
// -> bf16 gu (as the unfused GEMM stores them) and act = SiLU(g) * u from the
// rounded values (as the unfused act kernel computes it)
__device__ __forceinline__ void glu_fwd_chunk(const GemmParams& p, int row, int col0, const uint32_t (&vg)[32],
                                              const uint32_t (&vu)[32]) {
  __nv_bfloat16* grow = p.C + (int64_t)row * p.ldc + col0;
  __nv_bfloat16* urow = grow + p.glu_off;
  __nv_bfloat16* arow = p.aux + (int64_t)row * p.ld_aux + col0;
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    uint4 og, ou, oa;
    __nv_bfloat162* g2 = reinterpret_cast<__nv_bfloat162*>(&og);
    __nv_bfloat162* u2 = reinterpret_cast<__nv_bfloat162*>(&ou);
    __nv_bfloat162* a2 = reinterpret_cast<__nv_bfloat162*>(&oa);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      g2[t] = __floats2bfloat162_rn(__uint_as_float(vg[j + 2 * t]), __uint_as_float(vg[j + 2 * t + 1]));
      u2[t] = __floats2bfloat162_rn(__uint_as_float(vu[j + 2 * t]), __uint_as_float(vu[j + 2 * t + 1]));
      const float2 g = __bfloat1622float2(g2[t]), u = __bfloat1622float2(u2[t]);
      a2[t] = __floats2bfloat162_rn(silu_mul(g.x, u.x), silu_mul(g.y, u.y));
    }
    *reinterpret_cast<uint4*>(grow + j) = og;
    *reinterpret_cast<uint4*>(urow + j) = ou;
    *reinterpret_cast<uint4*>(arow + j) = oa;
  }
}

// GLU backward (mode 3): acc = dact (rounded to bf16 as the unfused GEMM
// stores it), g / u from gu -> d(gate), d(up) as the unfused act_bwd kernel
__device__ __forceinline__ void glu_bwd_chunk(const GemmParams& p, int row, int col0, const uint32_t (&v)[32]) {
  const __nv_bfloat16* gr = p.aux + (int64_t)row * p.ld_aux + col0;
  const __nv_bfloat16* ur = gr + p.glu_off;
  __nv_bfloat16* dgr = p.C + (int64_t)row * p.ldc + col0;
  __nv_bfloat16* dur = dgr + p.glu_off;
  // all eight 16-byte loads in flight before the first store (the stores could
  // alias them as far as the compiler knows, which would serialise the latency)
  uint4 gvs[4], uvs[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    gvs[t] = __ldg(reinterpret_cast<const uint4*>(gr) + t);
    uvs[t] = __ldg(reinterpret_cast<const uint4*>(ur) + t);
  }
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gvs[j / 8]);
    const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uvs[j / 8]);
    uint4 og, ou;
    __nv_bfloat162* dg2 = reinterpret_cast<__nv_bfloat162*>(&og);
    __nv_bfloat162* du2 = reinterpret_cast<__nv_bfloat162*>(&ou);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float2 g = __bfloat1622float2(g2[t]), u = __bfloat1622float2(u2[t]);
      const float da0 = __bfloat162float(__float2bfloat16_rn(__uint_as_float(v[j + 2 * t])));
      const float da1 = __bfloat162float(__float2bfloat16_rn(__uint_as_float(v[j + 2 * t + 1])));
      float dg0, du0, dg1, du1;
      silu_mul_bwd(da0, g.x, u.x, dg0, du0);
      silu_mul_bwd(da1, g.y, u.y, dg1, du1);
      dg2[t] = __floats2bfloat162_rn(dg0, dg1);
      du2[t] = __floats2bfloat162_rn(du0, du1);
    }
    *reinterpret_cast<uint4*>(dgr + j) = og;
    *reinterpret_cast<uint4*>(dur + j) = ou;
  }
}

template <int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
gemm_bf16_sm100(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB0,
                const __grid_constant__ CUtensorMap mapB1, const __grid_constant__ CUtensorMap mapB2,
                const __grid_constant__ CUtensorMap mapB3, const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(smB + STAGES * B_STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int num_tiles = p.m_tiles * p.n_tiles;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&mapA);
    ptx::tma_prefetch(&mapB0);
    if (p.nseg > 1) ptx::tma_prefetch(&mapB1);
    if (p.nseg > 2) ptx::tma_prefetch(&mapB2);
    if (p.nseg > 3) ptx::tma_prefetch(&mapB3);
    for (int s = 0; s < STAGES; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { ptx::mbar_init(&tfull[b], 1); ptx::mbar_init(&tempty[b], 4); }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ----------------------------------------------------------- producer
      int stage = 0; uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int mt, nt;
        tile_mn(p, tile, mt, nt);
        const int m0 = mt * BM;
        int bseg = 0, n0 = nt * BN;
        if (!p.split_k) {
          bseg = seg_of(p, nt);
          n0 = (nt - (bseg ? p.seg_end[bseg - 1] : 0)) * BN;
        }
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], A_STAGE + B_STAGE);
          uint8_t* a = smA + stage * A_STAGE;
          uint8_t* b = smB + stage * B_STAGE;
          const int k0 = kb * BK;
          if (!p.a_mn) {
            ptx::tma_load_2d(a, &mapA, &full[stage], k0, m0);
          } else {
            ptx::tma_load_2d(a, &mapA, &full[stage], m0, k0);
            ptx::tma_load_2d(a + 8192, &mapA, &full[stage], m0 + 64, k0);
          }
          int s = bseg, kk0 = k0;
          if (p.split_k) {
            s = seg_of(p, kb);
            kk0 = (kb - (s ? p.seg_end[s - 1] : 0)) * BK;
          }
          const CUtensorMap* mb = s == 0 ? &mapB0 : s == 1 ? &mapB1 : s == 2 ? &mapB2 : &mapB3;
          if (!p.b_mn) {
            ptx::tma_load_2d(b, mb, &full[stage], kk0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) ptx::tma_load_2d(b + j * 8192, mb, &full[stage], n0 + 64 * j, kk0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    // The whole warp walks the loop (warp-uniform descriptors stay in uniform
    // registers); one elected lane issues each tcgen05 instruction.
    const uint64_t a_d0 = p.a_mn ? ptx::umma_desc_sw128(ptx::smem_u32(smA), 8192, 1024)
                                 : ptx::umma_desc_sw128(ptx::smem_u32(smA), 16, 1024);
    const uint64_t b_d0 = p.b_mn ? ptx::umma_desc_sw128(ptx::smem_u32(smB), 8192, 1024)
                                 : ptx::umma_desc_sw128(ptx::smem_u32(smB), 16, 1024);
    const uint32_t a_ks = p.a_mn ? 2048 >> 4 : 32 >> 4;     // descriptor step per UMMA_K
    const uint32_t b_ks = p.b_mn ? 2048 >> 4 : 32 >> 4;
    int stage = 0; uint32_t phase = 0;
    int acc = 0; uint32_t aphase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      ptx::mbar_wait(&tempty[acc], aphase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d = tmem_base + acc * BN;
      for (int kb = 0; kb < p.k_blocks; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint64_t ad = a_d0 + (uint32_t)(stage * (A_STAGE >> 4));
        const uint64_t bd = b_d0 + (uint32_t)(stage * (B_STAGE >> 4));
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k)
            ptx::umma_f16(d, ad + k * a_ks, bd + k * b_ks, p.idesc, (kb | k) != 0);
          ptx::umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (ptx::elect_one()) ptx::umma_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------- epilogue
    const int q = warp & 3;
    int acc = 0; uint32_t aphase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int mt, nt;
        tile_mn(p, tile, mt, nt);
      ptx::mbar_wait(&tfull[acc], aphase);
      ptx::tc_fence_after();
      const int row = mt * BM + q * 32 + lane;
      const bool row_ok = row < p.M;
      __nv_bfloat16* crow = p.C + (int64_t)row * p.ldc;
      const __nv_bfloat16* rrow = p.R ? p.R + (int64_t)row * p.ldr : nullptr;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, v);
        ptx::tmem_ld_wait();
        const int col0 = nt * BN + c * 32;
        if (row_ok && col0 < p.N) {
          if constexpr (EPI == 1) {
            epilogue_chunk<1>(p, row, col0, v);
          } else {
            float f[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
            if (rrow) {
              if (col0 + 32 <= p.N) {
#pragma unroll
                for (int j = 0; j < 32; j += 8) {
                  uint4 rv = *reinterpret_cast<const uint4*>(rrow + col0 + j);
                  const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&rv);
#pragma unroll
                  for (int t = 0; t < 4; ++t) {
                    float2 rf = __bfloat1622float2(r2[t]);
                    f[j + 2 * t] = __fadd_rn(f[j + 2 * t], rf.x);
                    f[j + 2 * t + 1] = __fadd_rn(f[j + 2 * t + 1], rf.y);
                  }
                }
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (col0 + j < p.N) f[j] = __fadd_rn(f[j], __bfloat162float(rrow[col0 + j]));
              }
            }
            if (col0 + 32 <= p.N) {
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                uint4 o;
                __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
                for (int t = 0; t < 4; ++t) o2[t] = __floats2bfloat162_rn(f[j + 2 * t], f[j + 2 * t + 1]);
                *reinterpret_cast<uint4*>(crow + col0 + j) = o;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (col0 + j < p.N) crow[col0 + j] = __float2bfloat16_rn(f[j]);
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  }
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ------------------------------------------------------------------ GEMM side job
constexpr int SIDE_WARPS = 6;               // warps 2, 3, 8, 9, 10, 11 of the pair kernel
__device__ __forceinline__ void side_job(const SideJob& sj, int side_warp, int lane) {
  const int64_t nthr = (int64_t)gridDim.x * SIDE_WARPS * 32;
  const int64_t t = (int64_t)blockIdx.x * SIDE_WARPS * 32 + side_warp * 32 + lane;
  const uint64_t pol = policy_evict_first();
  const AdamScalars a = adam_scalars(sj.w1, sj.w2, sj.b2, sj.neg_s, sj.c, sj.eps, 1.0f);
  for (int64_t g = sj.g0 + t; g < sj.g1; g += 2 * nthr) {
    Group8<1> x[2];
    int mi[2];
    int64_t j[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {          // both groups' loads before any math
      const int64_t gg = g + u * nthr;
      mi[u] = 0;
      for (int i = 1; i < sj.nm; ++i)
        if (gg >= sj.cum[i]) mi[u] = i;
      j[u] = gg - sj.cum[mi[u]];
      if (gg < sj.g1) {
        const uint8_t* gp = sj.slot + sj.goff[mi[u]] + j[u] * 16;
        const int64_t e = sj.store_off[mi[u]] + 8 * j[u];
        load_group8<1>(x[u], &gp, 1, sj.master + e, sj.m + e, sj.v + e, pol);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (g + u * nthr < sj.g1) {
        const int64_t e = sj.store_off[mi[u]] + 8 * j[u];
        finish_group8<1>(x[u], 1, sj.master + e, sj.m + e, sj.v + e, sj.shard + e, a, pol);
      }
    }
  }
}

// ------------------------------------------------------------------ CTA-pair kernel
// cta_group::2: a cluster of 2 CTAs on one TPC computes a 256 x 256 tile.  CTA
// r stages rows [128r, 128r+128) of A and columns [128r, 128r+128) of B (16 KiB
// each per 64-deep K block), so each SM moves half the operand bytes of the
// 1-CTA kernel per MMA; 6 stages fit in 192 KiB.  The leader (rank 0) issues
// tcgen05.mma.cta_group::2 (M = 256) and commits, multicast to both CTAs, the
// smem-slot release and the accumulator-ready barriers.  Each CTA's TMEM holds
// its 128 rows x 256 fp32 columns (x2 buffers = 512 columns).
constexpr int BM2 = 256;
constexpr int A2_STAGE = 128 * BK * 2;        // 16 KiB per CTA
template <int BNT, int ST> struct Pair {
  static constexpr int B_STAGE = (BNT / 2) * BK * 2;                    // B half per CTA
  static constexpr int STAGES = ST;                                      // <= 7 @256, <= 9 @128
  static_assert(ST * (A2_STAGE + B_STAGE) + 1280 <= 227 * 1024, "smem");
  static constexpr int SMEM = STAGES * (A2_STAGE + B_STAGE) + 1024 + 256;
  static constexpr int TMEM = 2 * BNT;                                   // 2 accumulator buffers
};

constexpr int GEMM2_THREADS = 384;          // + side-job warps 8..11

// CW: per-tile chunk waits of a fused all-gather (dc_gemm_args.chunk_*); a
// separate instantiation, so the default kernels carry none of that code
// (r02: even the untaken branch and its call made the step ~6 % slower)
// HT: half-width tail units (p.ht_on), also a separate instantiation
template <int BNT, int ST, int EPI, bool CW = false, bool HT = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM2_THREADS, 1)
gemm2_bf16_sm100(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB0,
                 const __grid_constant__ CUtensorMap mapB1, const __grid_constant__ CUtensorMap mapB2,
                 const __grid_constant__ CUtensorMap mapB3, const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* smA = smem;
  uint8_t* smB = smem + Pair<BNT, ST>::STAGES * A2_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(smB + Pair<BNT, ST>::STAGES * Pair<BNT, ST>::B_STAGE);
  uint64_t* empty = full + Pair<BNT, ST>::STAGES;
  uint64_t* tfull = empty + Pair<BNT, ST>::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  [[maybe_unused]] uint32_t* cw_progress = tmem_slot + 1;   // CW: B loads the watcher has cleared
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
  const WorkList wl = work_list<HT>(p, pair, npairs);
  const int nunits = wl.count();

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&mapA);
    ptx::tma_prefetch(&mapB0);
    if (p.nseg > 1) ptx::tma_prefetch(&mapB1);
    if (p.nseg > 2) ptx::tma_prefetch(&mapB2);
    if (p.nseg > 3) ptx::tma_prefetch(&mapB3);
    for (int s = 0; s < Pair<BNT, ST>::STAGES; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { ptx::mbar_init(&tfull[b], 1); ptx::mbar_init(&tempty[b], 8); }
    if constexpr (CW) *cw_progress = 0u;
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm(tmem_slot, Pair<BNT, ST>::TMEM);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ----------------------------------------------------------- producer (both CTAs)
      int stage = 0; uint32_t phase = 0;
      [[maybe_unused]] int cw_step = 0;               // chunk waits: this load's index in the watcher's walk
      for (int ui = 0; ui < nunits; ++ui) {
        const Unit un = unit_at<HT>(p, wl, pair, npairs, ui);
        const int tile = un.tile;
        int mt, nt;
        tile_mn(p, tile, mt, nt);
        const int m0 = mt * BM2 + (int)rank * 128;
        int bseg = 0, n0 = nt * BNT;
        if constexpr (EPI == 2) {            // GLU: CTA r stages segment r (gate | up), same columns
          bseg = (int)rank;
          n0 = nt * (BNT / 2);
        } else {
          if (!p.split_k) {
            bseg = seg_of(p, nt);
            n0 = (nt - (bseg ? p.seg_end[bseg - 1] : 0)) * BNT;
          }
          if constexpr (HT)    // half tile: columns [half 128, half 128 + 128) of the tile, 64 per CTA
            n0 += un.half < 0 ? (int)rank * (BNT / 2) : un.half * (BNT / 2) + (int)rank * (BNT / 4);
          else
            n0 += (int)rank * (BNT / 2);
        }
        // an MN-major half tile loads one 64-column box per CTA instead of two
        uint32_t b_bytes = Pair<BNT, ST>::B_STAGE;
        if constexpr (HT) b_bytes = (un.half >= 0 && p.b_mn) ? Pair<BNT, ST>::B_STAGE / 2 : Pair<BNT, ST>::B_STAGE;
        for (int kb = un.kb0; kb < un.kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], 2 * (A2_STAGE + b_bytes));
          const uint32_t lbar = ptx::mapa(ptx::smem_u32(&full[stage]), 0);
          uint8_t* a = smA + stage * A2_STAGE;
          uint8_t* b = smB + stage * Pair<BNT, ST>::B_STAGE;
          const int k0 = kb * BK;
          if (!p.a_mn) {
            ptx::tma_load_2d_2sm(a, &mapA, lbar, k0, m0);
          } else {
            ptx::tma_load_2d_2sm(a, &mapA, lbar, m0, k0);
            ptx::tma_load_2d_2sm(a + 8192, &mapA, lbar, m0 + 64, k0);
          }
          int s = bseg, kk0 = k0;
          if (p.split_k) {
            s = seg_of(p, kb);
            kk0 = (kb - (s ? p.seg_end[s - 1] : 0)) * BK;
          }
          const CUtensorMap* mb = s == 0 ? &mapB0 : s == 1 ? &mapB1 : s == 2 ? &mapB2 : &mapB3;
          if constexpr (CW) {  // fused all-gather: the watcher (warp 3) has seen this load's chunks land
            while (ld_acquire_cta(cw_progress) <= (uint32_t)cw_step) __nanosleep(32);
            asm volatile("fence.proxy.async.global;" ::: "memory");   // peer (generic) stores -> TMA reads
            ++cw_step;
          }
          if (!p.b_mn) {
            ptx::tma_load_2d_2sm(b, mb, lbar, kk0, n0);
          } else if constexpr (HT) {
            const int nbox = un.half < 0 ? BNT / 128 : BNT / 256;
            for (int j = 0; j < nbox; ++j) ptx::tma_load_2d_2sm(b + j * 8192, mb, lbar, n0 + 64 * j, kk0);
          } else {
#pragma unroll
            for (int j = 0; j < BNT / 128; ++j) ptx::tma_load_2d_2sm(b + j * 8192, mb, lbar, n0 + 64 * j, kk0);
          }
          if (++stage == Pair<BNT, ST>::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ----------------------------------------------------------- MMA issuer (leader CTA)
      // whole warp walks the loop (uniform descriptors); one elected lane issues
      const uint64_t a_d0 = p.a_mn ? ptx::umma_desc_sw128(ptx::smem_u32(smA), 8192, 1024)
                                   : ptx::umma_desc_sw128(ptx::smem_u32(smA), 16, 1024);
      const uint64_t b_d0 = p.b_mn ? ptx::umma_desc_sw128(ptx::smem_u32(smB), 8192, 1024)
                                   : ptx::umma_desc_sw128(ptx::smem_u32(smB), 16, 1024);
      const uint32_t a_ks = p.a_mn ? 2048 >> 4 : 32 >> 4;
      const uint32_t b_ks = p.b_mn ? 2048 >> 4 : 32 >> 4;
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t aphase = 0;
      for (int ui = 0; ui < nunits; ++ui) {
        const Unit un = unit_at<HT>(p, wl, pair, npairs, ui);
        ptx::mbar_wait(&tempty[acc], aphase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + acc * BNT;
        for (int kb = un.kb0; kb < un.kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint64_t ad = a_d0 + (uint32_t)(stage * (A2_STAGE >> 4));
          const uint64_t bd = b_d0 + (uint32_t)(stage * (Pair<BNT, ST>::B_STAGE >> 4));
          if (ptx::elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k)
              ptx::umma_f16_2sm(d, ad + k * a_ks, bd + k * b_ks, (HT && un.half >= 0) ? p.idesc_half : p.idesc,
                                (kb != un.kb0) | (k != 0));
            ptx::umma_commit_2sm_mc(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == Pair<BNT, ST>::STAGES) { stage = 0; phase ^= 1; }
        }
        if (ptx::elect_one()) ptx::umma_commit_2sm_mc(&tfull[acc], 0x3);
        __syncwarp();
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
    }
  } else if (CW && warp == 3) {   // (warp 3 is a side-job warp otherwise)
    if constexpr (CW) {
      {
        // ------------------------------------------------------- chunk watcher (fused all-gather)
        // Walks the producer's sequence of B loads ahead of it; for each one
        // waits (acquire, system scope) until the gather chunks it reads have
        // landed and then publishes the count of cleared loads in shared
        // memory, so the system-scope flag latency stays off the producer's
        // critical path.  A verified chunk range is cached (end of the last
        // chunk seen), so consecutive k-blocks / tiles rarely touch a flag.
        int v_seg = -1;
        int64_t v_lo = 0, v_hi = 0;
        uint32_t n = 0;
        for (int ui = 0; ui < nunits; ++ui) {
          const Unit un = unit_at<HT>(p, wl, pair, npairs, ui);
          int mt, nt;
          tile_mn(p, un.tile, mt, nt);
          int bseg = 0, n0 = nt * BNT;
          if constexpr (EPI == 2) {
            bseg = (int)rank;
            n0 = nt * (BNT / 2);
          } else {
            if (!p.split_k) {
              bseg = seg_of(p, nt);
              n0 = (nt - (bseg ? p.seg_end[bseg - 1] : 0)) * BNT;
            }
            n0 += (int)rank * (BNT / 2);
          }
          for (int kb = un.kb0; kb < un.kb1; ++kb) {
            int sg = bseg, kk0 = kb * BK;
            if (p.split_k) {
              sg = seg_of(p, kb);
              kk0 = (kb - (sg ? p.seg_end[sg - 1] : 0)) * BK;
            }
            if (p.cf[sg]) {
              const int64_t e0 = p.b_mn ? (int64_t)kk0 * p.cld[sg] + n0 : (int64_t)n0 * p.cld[sg];
              const int64_t e1 = p.b_mn ? (int64_t)(kk0 + BK - 1) * p.cld[sg] + n0 + BNT / 2
                                        : (int64_t)(n0 + BNT / 2) * p.cld[sg];
              if (sg != v_seg || e0 < v_lo || e1 > v_hi) {
                const bool extend = sg == v_seg && e0 >= v_lo && e0 <= v_hi;
                const int64_t from = extend ? v_hi : e0;
                const int64_t end = chunk_wait(p.cf[sg], p.cS[sg], p.cE[sg], p.cn[sg], p.cval[sg], p.cerr, p.ctmo,
                                               from, e1);
                if (extend) v_hi = end;
                else { v_seg = sg; v_lo = e0; v_hi = end; }
              }
            }
            ++n;
            __syncwarp();
            if (lane == 0) st_release_cta(cw_progress, n);
          }
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------- epilogue (both CTAs)
    const int q = warp & 3;
    const int rl = q * 32 + lane;                 // this thread's row inside the CTA's 128
    int acc = 0; uint32_t aphase = 0;
    for (int ui = 0; ui < nunits; ++ui) {
      const Unit un = unit_at<HT>(p, wl, pair, npairs, ui);
      const int tile = un.tile;
      int mt, nt;
        tile_mn(p, tile, mt, nt);
      // split tile: fp32 partial of this CTA's 128 rows, [chunk][j/4][row][4]
      float* ws = un.mode ? p.sk_ws + ((int64_t)(tile - p.sk_dp) * 2 + rank) * (128 * BNT) : nullptr;
      uint32_t* flag = un.mode ? p.sk_flags + (tile - p.sk_dp) * 2 + rank : nullptr;
      if (un.mode == 2) {                          // the head's partial must have landed
        const uint64_t t0 = ptx::globaltimer();
        while (ptx::ld_acquire_gpu(flag) != p.sk_epoch)
          if (ptx::globaltimer() - t0 > 4000000000ull) __trap();
      }
      ptx::mbar_wait(&tfull[acc], aphase);
      ptx::tc_fence_after();
      const int row = mt * BM2 + (int)rank * 128 + rl;
      const bool row_ok = row < p.M;
      __nv_bfloat16* crow = p.C + (int64_t)row * p.ldc;
      const __nv_bfloat16* rrow = p.R ? p.R + (int64_t)row * p.ldr : nullptr;
      if constexpr (EPI == 2) {
        // GLU forward: accumulator columns [0, BNT/2) = gate, [BNT/2, BNT) = up
#pragma unroll 1
        for (int c = 0; c < BNT / 64; ++c) {
          uint32_t vg[32], vu[32];
          ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BNT + c * 32, vg);
          ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BNT + BNT / 2 + c * 32, vu);
          ptx::tmem_ld_wait();
          const int col0 = nt * (BNT / 2) + c * 32;
          if (row_ok && col0 < p.N) glu_fwd_chunk(p, row, col0, vg, vu);
        }
      }
      int nchunk = EPI == 2 ? 0 : BNT / 32, colh = 0;
      if constexpr (HT) {
        if (un.half >= 0) { nchunk = BNT / 64; colh = un.half * (BNT / 2); }
      }
#pragma unroll 1
      for (int c = 0; c < nchunk; ++c) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BNT + c * 32, v);
        ptx::tmem_ld_wait();
        const int col0 = nt * BNT + colh + c * 32;
        if (un.mode == 1) {                        // head: store the raw fp32 partial
          float4* w4 = reinterpret_cast<float4*>(ws) + (int64_t)c * 8 * 128 + rl;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            __stcg(w4 + j * 128, make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                             __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3])));
          continue;
        }
        if (un.mode == 2) {                        // tail: partial(head) + this part, fp32
          const float4* w4 = reinterpret_cast<const float4*>(ws) + (int64_t)c * 8 * 128 + rl;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 h = __ldcg(w4 + j * 128);
            v[4 * j] = __float_as_uint(__fadd_rn(h.x, __uint_as_float(v[4 * j])));
            v[4 * j + 1] = __float_as_uint(__fadd_rn(h.y, __uint_as_float(v[4 * j + 1])));
            v[4 * j + 2] = __float_as_uint(__fadd_rn(h.z, __uint_as_float(v[4 * j + 2])));
            v[4 * j + 3] = __float_as_uint(__fadd_rn(h.w, __uint_as_float(v[4 * j + 3])));
          }
        }
        if (row_ok && col0 < p.N) {
          if constexpr (EPI == 1) {
            epilogue_chunk<1>(p, row, col0, v);
          } else if constexpr (EPI == 3) {
            glu_bwd_chunk(p, row, col0, v);
          } else {
            float f[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
            if (rrow) {
              if (col0 + 32 <= p.N) {
#pragma unroll
                for (int j = 0; j < 32; j += 8) {
                  uint4 rv = *reinterpret_cast<const uint4*>(rrow + col0 + j);
                  const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&rv);
#pragma unroll
                  for (int t = 0; t < 4; ++t) {
                    float2 rf = __bfloat1622float2(r2[t]);
                    f[j + 2 * t] = __fadd_rn(f[j + 2 * t], rf.x);
                    f[j + 2 * t + 1] = __fadd_rn(f[j + 2 * t + 1], rf.y);
                  }
                }
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (col0 + j < p.N) f[j] = __fadd_rn(f[j], __bfloat162float(rrow[col0 + j]));
              }
            }
            if (col0 + 32 <= p.N) {
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                uint4 o;
                __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
                for (int t = 0; t < 4; ++t) o2[t] = __floats2bfloat162_rn(f[j + 2 * t], f[j + 2 * t + 1]);
                *reinterpret_cast<uint4*>(crow + col0 + j) = o;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (col0 + j < p.N) crow[col0 + j] = __float2bfloat16_rn(f[j]);
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
      if (un.mode == 1) {                          // publish the partial (all 128 rows written)
        __threadfence();
        ptx::named_bar_sync(1, 128);
        if (rl == 0) ptx::st_release_gpu(flag, p.sk_epoch);
      }
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  } else if (p.side.nm > 0) {
    // ------------------------------------------------------------- side job (warps 2, 3, 8..11)
    side_job(p.side, warp < 4 ? warp - 2 : warp - 6, lane);
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm(tmem_base, Pair<BNT, ST>::TMEM);
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// 2-D bf16 tensor map: inner dimension `inner` (contiguous) x `outer` rows,
// row pitch `ld` elements, box {64, box_outer}, 128-byte swizzle, OOB -> 0.
static bool make_map(CUtensorMap* m, const void* ptr, int64_t inner, int64_t outer, int64_t ld,
                     int box_outer) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int num_sms_cached() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// stream-K workspace: caller-owned (dc_gemm_args.workspace), [tiles_cap][2]
// CTA partials of 128 x 256 fp32, then [tiles_cap][2] uint32 flags.  The
// launch epoch of each workspace is kept here, keyed by its address: a flag
// equal to the current epoch marks a partial of the current launch.
constexpr size_t SK_TILES_CAP = 2 * 74 + 2, SK_PART_BYTES = 2ull * 128 * 256 * 4;
constexpr size_t SK_FLAG_BYTES = SK_TILES_CAP * 2 * 4;
constexpr size_t SK_WS_BYTES = SK_TILES_CAP * SK_PART_BYTES + SK_FLAG_BYTES;
static std::mutex g_sk_mu;
static std::map<const void*, uint32_t> g_sk_epoch;
static uint32_t sk_next_epoch(const void* ws) {
  std::lock_guard<std::mutex> lock(g_sk_mu);
  return ++g_sk_epoch[ws];
}

// graph mode: a step starts from epoch 0 with cleared flags, so the epochs a
// replayed graph baked in at capture never meet a previous replay's flags
void gemm_sk_reset(void* ws, cudaStream_t st) {
  if (!ws) return;
  std::lock_guard<std::mutex> lock(g_sk_mu);
  cudaMemsetAsync(reinterpret_cast<uint8_t*>(ws) + SK_TILES_CAP * SK_PART_BYTES, 0, SK_FLAG_BYTES, st);
  g_sk_epoch[ws] = 0;
}
uint64_t gemm_workspace_bytes() { return SK_WS_BYTES; }

// 0: 256-wide 6 stages (default), 2: 256-wide 7 stages (DC_GEMM_STAGES=7)
static int env_st_pick() {
  static const int v = (getenv("DC_GEMM_STAGES") && atoi(getenv("DC_GEMM_STAGES")) == 7) ? 2 : 0;
  return v;
}

// co-resident 2-CTA clusters of a pair-kernel configuration (0: 256/6, 1: 128/9,
// 2: 256/7), from cudaOccupancyMaxActiveClusters; filled by preload
static int g_pair_slots[3] = {0, 0, 0};
static int pair_slots(int cfg) { return g_pair_slots[cfg]; }

template <int BN_, int ST_>
static cudaError_t query_pair_slots(int* out) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * 148, 1, 1);
  cfg.blockDim = dim3(GEMM2_THREADS, 1, 1);
  cfg.dynamicSmemBytes = Pair<BN_, ST_>::SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(out, gemm2_bf16_sm100<BN_, ST_, 0>, &cfg);
}

dc_status launch_gemm(const dc_gemm_args* g, cudaStream_t stream, std::string* err, const EpiAdam* adam,
                      const SideJob* side) {
  if (g->M <= 0 || g->N <= 0 || g->K <= 0 || (g->N % 8) || (g->K % 8) || g->n_bseg < 1 || g->n_bseg > 4) {
    *err = "dc_gemm: M,N,K must be > 0, N and K multiples of 8, 1..4 B segments";
    return DC_EINVAL;
  }
  static const int env_sms = getenv("DC_GEMM_SMS") ? atoi(getenv("DC_GEMM_SMS")) : 0;
  static const int env_kernel = getenv("DC_GEMM_KERNEL") ? atoi(getenv("DC_GEMM_KERNEL")) : 0;
  int sms = g->num_sms > 0 ? g->num_sms : (env_sms > 0 ? env_sms : num_sms_cached());
  const int kind = g->kernel ? g->kernel : (env_kernel ? env_kernel : 2);
  const bool pair = kind == 2 && sms >= 2;
  const int tm = pair ? BM2 : BM;                // tile rows
  // pair tile width: 256 unless 128 wastes clearly less of the last wave
  int bnt = BN;
  if (pair) {
    const int pairs = sms / 2;
    const int64_t mt = (g->M + BM2 - 1) / BM2;
    auto eff = [&](int bn) {
      const int64_t t = mt * ((g->N + bn - 1) / bn);
      const int64_t waves = (t + pairs - 1) / pairs;
      return (double)t / (double)(waves * pairs);
    };
    const int forced = getenv("DC_GEMM_BN") ? atoi(getenv("DC_GEMM_BN")) : 0;
    if (forced == 128 || forced == 256) bnt = forced;
    (void)eff;   // 256 x 128 pair tiles measured slower on every layer shape (r01); forced only
  }
  const int rows_per_cta = 128;                  // A rows / B cols staged by one CTA
  GemmParams p{};
  p.M = g->M; p.N = g->N; p.K = g->K;
  p.m_tiles = (g->M + tm - 1) / tm;
  p.n_tiles = (g->N + bnt - 1) / bnt;
  p.k_blocks = (g->K + BK - 1) / BK;
  p.nseg = g->n_bseg; p.split_k = g->b_split_k;
  p.a_mn = g->a_mn_major; p.b_mn = g->b_mn_major;
  p.C = reinterpret_cast<__nv_bfloat16*>(g->C); p.ldc = g->ldc;
  p.R = reinterpret_cast<const __nv_bfloat16*>(g->R); p.ldr = g->ldr;
  if (adam) {
    if (g->ldc != g->N || g->R) { *err = "dc_gemm: fused Adam epilogue needs ldc == N and no residual"; return DC_EINVAL; }
    p.epi = 1;
    p.master = adam->master; p.m = adam->m; p.v = adam->v;
    p.shard = reinterpret_cast<__nv_bfloat16*>(adam->shard);
    p.w1 = adam->w1; p.w2 = adam->w2; p.b2 = adam->b2; p.neg_s = adam->neg_s; p.c = adam->c; p.eps = adam->eps;
  }
  if (side && side->nm > 0) {
    if (!pair) { *err = "dc_gemm: a side job needs the CTA-pair kernel"; return DC_EINVAL; }
    p.side = *side;
  }
  for (int s = 0; s < g->n_bseg; ++s) {
    if (!g->chunk_flags[s]) continue;
    if (!pair || g->chunk_S[s] < 8 || g->chunk_E[s] < 8 || g->chunk_numel[s] < 1 ||
        (g->chunk_S[s] + g->chunk_E[s] - 1) / g->chunk_E[s] > AG_CHUNKS)
      { *err = "dc_gemm: chunk waits need the CTA-pair kernel, S, E >= 8 and at most 64 chunks per shard"; return DC_EINVAL; }
    p.cf[s] = g->chunk_flags[s];
    p.cS[s] = g->chunk_S[s]; p.cE[s] = g->chunk_E[s]; p.cn[s] = g->chunk_numel[s];
    p.cld[s] = g->ldb[s];
    p.cval[s] = g->chunk_value[s];
  }
  p.cerr = g->chunk_err;
  p.ctmo = g->chunk_timeout_ns ? g->chunk_timeout_ns : 20ull * 1000 * 1000 * 1000;
  const int glu = g->epilogue;
  if (glu) {
    if (glu != 2 && glu != 3) { *err = "dc_gemm: epilogue is 0, 2 or 3"; return DC_EINVAL; }
    if (!pair || bnt != 256 || adam || (side && side->nm > 0) || g->R || !g->aux || (g->N % 128) ||
        (g->ld_aux % 8) || (g->glu_off % 8) || (g->ldc % 8))
      { *err = "dc_gemm: GLU epilogue needs the 256-wide pair kernel, N % 128 == 0, aux, 16 B aligned rows, no R"; return DC_EINVAL; }
    if (glu == 2 && (g->n_bseg != 2 || g->b_split_k || g->b_mn_major))
      { *err = "dc_gemm: GLU forward needs B = {gate, up}, K-major, split along N"; return DC_EINVAL; }
    p.epi = glu;
    p.aux = reinterpret_cast<__nv_bfloat16*>(g->aux);
    p.ld_aux = g->ld_aux;
    p.glu_off = g->glu_off;
    if (glu == 2) p.n_tiles = (g->N + 127) / 128;     // a tile = 128 gate + the same 128 up columns
  }
  p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)p.a_mn << 15) | ((uint32_t)p.b_mn << 16) |
            ((uint32_t)(bnt >> 3) << 17) | ((uint32_t)(tm >> 4) << 24);
  CUtensorMap mA, mB[4];
  bool ok = p.a_mn ? make_map(&mA, g->A, g->M, g->K, g->lda, 64)
                   : make_map(&mA, g->A, g->K, g->M, g->lda, rows_per_cta);
  int prev = 0;
  for (int s = 0; s < g->n_bseg && glu == 2; ++s)   // GLU: two [N][K] K-major tensors, CTA r reads segment r
    ok = ok && make_map(&mB[s], g->B[s], g->K, g->N, g->ldb[s], bnt / 2);
  for (int s = 0; s < g->n_bseg && glu != 2; ++s) {
    p.seg_end[s] = g->bseg_end[s];
    const int unit = g->b_split_k ? BK : BN;
    const int64_t lo = (int64_t)prev * unit;
    int64_t hi = (int64_t)g->bseg_end[s] * unit;
    const int64_t full_ext = g->b_split_k ? g->K : g->N;
    if (s == g->n_bseg - 1) hi = full_ext;
    if (hi > full_ext) hi = full_ext;
    if (hi <= lo) { *err = "dc_gemm: empty or unordered B segment"; return DC_EINVAL; }
    const int64_t ext = hi - lo;                   // this segment's N (or K) extent
    const int64_t kdim = g->b_split_k ? ext : g->K;
    const int64_t ndim = g->b_split_k ? g->N : ext;
    ok = ok && (g->b_mn_major ? make_map(&mB[s], g->B[s], ndim, kdim, g->ldb[s], 64)
                              : make_map(&mB[s], g->B[s], kdim, ndim, g->ldb[s], pair ? bnt / 2 : BN));
    prev = g->bseg_end[s];
  }
  if (!g->b_split_k && glu != 2)   // caller's N segment ends are in units of 256 columns
    for (int s = 0; s < g->n_bseg; ++s) p.seg_end[s] *= 256 / bnt;
  if (g->n_bseg == 1) p.seg_end[0] = g->b_split_k ? p.k_blocks : p.n_tiles;
  for (int s = g->n_bseg; s < 4; ++s) { mB[s] = mB[0]; p.seg_end[s] = p.seg_end[g->n_bseg - 1]; }
  if (!ok) { *err = "dc_gemm: cuTensorMapEncodeTiled failed (alignment / pitch must be 16 B)"; return DC_EINVAL; }
  static std::once_flag attr_once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once, [] { attr_err = preload_gemm_kernels(); });
  if (attr_err != cudaSuccess) {
    *err = std::string("dc_gemm: kernel setup failed: ") + cudaGetErrorString(attr_err);
    return DC_ECUDA;
  }
  const int tiles = p.m_tiles * p.n_tiles;
  {   // tile order: groups of DC_GEMM_GROUP_DEFAULT (2) m-tiles when m_tiles >= 2 n_tiles
      // (profiles/r01g/gemm_group/: the 56 x 16-tile gate / up dW GEMMs read 0.18 instead of 1.3 GB
      // of DRAM and run 10 % faster; grouping the wide forward GEMMs would re-stream B per group
      // instead).  DC_GEMM_GROUP_M overrides for every GEMM (0: never group).
    static const int env_g = getenv("DC_GEMM_GROUP_M") ? atoi(getenv("DC_GEMM_GROUP_M")) : -1;
    const int auto_g = p.m_tiles >= 2 * p.n_tiles ? DC_GEMM_GROUP_DEFAULT : 0;
    const int gsz = g->tile_group_m > 0 ? g->tile_group_m : g->tile_group_m < 0 ? 0 : env_g < 0 ? auto_g : env_g;
    p.group_m = (gsz > 0 && gsz < p.m_tiles) ? gsz : p.m_tiles;
  }
  if (pair) {
    // persistent grid: never more pairs than can be co-resident (an odd SM
    // count in a GPC leaves an SM without a partner; a non-resident pair
    // would run as a second wave after the others finished)
    const int slots = pair_slots(bnt == 128 ? 1 : env_st_pick());
    const int pairs = std::min(tiles, std::min(sms / 2, slots > 0 ? slots : sms / 2));
    static const bool sk_env = !(getenv("DC_GEMM_SK") && atoi(getenv("DC_GEMM_SK")) == 0);
    static const int sk_min_kb = getenv("DC_GEMM_SK_MINKB") ? atoi(getenv("DC_GEMM_SK_MINKB")) : 128;   // A/B knob
    // stream-K pays only when the k-loop is long (measured on the layer shapes,
    // profiles/r01d: +3-4 % at K >= 14336, -2 % at K = 4096, where the idle
    // pairs of the last partial wave let the others clock higher)
    if (g->stream_k && g->workspace && sk_env && !p.epi && tiles > pairs && tiles % pairs && p.k_blocks >= sk_min_kb &&
        tiles - (tiles / pairs - 1) * pairs <= 150) {
      if (g->workspace_bytes < SK_WS_BYTES || (reinterpret_cast<uintptr_t>(g->workspace) & 255))
        { *err = "dc_gemm: stream-K workspace smaller than dc_gemm_workspace_bytes() or not 256 B aligned"; return DC_EINVAL; }
      p.sk_on = 1;
      p.sk_dp = (tiles / pairs - 1) * pairs;            // leaves [pairs, 2 pairs) tiles to split
      p.sk_total = (int64_t)(tiles - p.sk_dp) * p.k_blocks;
      p.sk_ws = reinterpret_cast<float*>(g->workspace);
      p.sk_flags = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(g->workspace) + SK_TILES_CAP * SK_PART_BYTES);
      p.sk_epoch = sk_next_epoch(g->workspace);
    }
    bool cw = false;
    for (int s = 0; s < 4; ++s) cw = cw || p.cf[s];
    {   // half-width tail units when the partial last wave fits in one wave of halves; forward-form
        // GEMMs only (A and B K-major): measured in-step, the dX / dW GEMMs of the backward (which
        // share the device with each other, dw_concurrent) got 7-25 % slower with them, the
        // forward ones 1-7 % faster (profiles/r02/half_tail/)
      static const int ht_env = getenv("DC_GEMM_HALF_TAIL") ? atoi(getenv("DC_GEMM_HALF_TAIL")) : 1;
      const int dp = tiles / pairs * pairs;
      if (ht_env && bnt == 256 && !p.sk_on && !p.epi && !cw && !(side && side->nm > 0) && tiles > pairs &&
          !p.a_mn && !p.b_mn &&
          tiles > dp && 2 * (tiles - dp) <= pairs) {
        p.ht_on = 1;
        p.ht_dp = dp;
        p.idesc_half = (p.idesc & ~(0x3Fu << 17)) | ((uint32_t)(128 >> 3) << 17);
      }
    }
    const int env_st = glu ? 6 : (env_st_pick() == 2 ? 7 : 6);
    const int g2 = 2 * pairs;
#define DC_PAIR_LAUNCH(BN_, ST_)                                                                   \
    (p.epi ? gemm2_bf16_sm100<BN_, ST_, 1><<<g2, GEMM2_THREADS, Pair<BN_, ST_>::SMEM, stream>>>(mA, mB[0], mB[1], mB[2], mB[3], p) \
           : gemm2_bf16_sm100<BN_, ST_, 0><<<g2, GEMM2_THREADS, Pair<BN_, ST_>::SMEM, stream>>>(mA, mB[0], mB[1], mB[2], mB[3], p))
    if (cw && (bnt != 256 || (p.epi != 0 && p.epi != 2)))
      { *err = "dc_gemm: chunk waits need the 256-wide pair kernel with epilogue 0 or 2"; return DC_EINVAL; }
    if (cw && glu == 2) gemm2_bf16_sm100<256, 6, 2, true><<<g2, GEMM2_THREADS, Pair<256, 6>::SMEM, stream>>>(mA, mB[0], mB[1], mB[2], mB[3], p);
    else if (cw) gemm2_bf16_sm100<256, 6, 0, true><<<g2, GEMM2_THREADS, Pair<256, 6>::SMEM, stream>>>(mA, mB[0], mB[1], mB[2], mB[3], p);
    else if (glu == 2) gemm2_bf16_sm100<256, 6, 2><<<g2, GEMM2_THREADS, Pair<256, 6>::SMEM, stream>>>(mA, mB[0], mB[1], mB[2], mB[3], p);
    else if (glu == 3) gemm2_bf16_sm100<256, 6, 3><<<g2, GEMM2_THREADS, Pair<256, 6>::SMEM, stream>>>(mA, mB[0], mB[1], mB[2], mB[3], p);
    else if (p.ht_on && env_st == 6)
      gemm2_bf16_sm100<256, 6, 0, false, true><<<g2, GEMM2_THREADS, Pair<256, 6>::SMEM, stream>>>(mA, mB[0], mB[1], mB[2], mB[3], p);
    else if (p.ht_on)
      gemm2_bf16_sm100<256, 7, 0, false, true><<<g2, GEMM2_THREADS, Pair<256, 7>::SMEM, stream>>>(mA, mB[0], mB[1], mB[2], mB[3], p);
    else if (bnt == 128) DC_PAIR_LAUNCH(128, 9);
    else if (env_st == 6) DC_PAIR_LAUNCH(256, 6);
    else DC_PAIR_LAUNCH(256, 7);
#undef DC_PAIR_LAUNCH
  } else {
    const int grid = tiles < sms ? tiles : sms;
    if (p.epi) gemm_bf16_sm100<1><<<grid, GEMM_THREADS, GEMM_SMEM, stream>>>(mA, mB[0], mB[1], mB[2], mB[3], p);
    else gemm_bf16_sm100<0><<<grid, GEMM_THREADS, GEMM_SMEM, stream>>>(mA, mB[0], mB[1], mB[2], mB[3], p);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { *err = std::string("dc_gemm launch: ") + cudaGetErrorString(e); return DC_ECUDA; }
  count_launch();
  return DC_OK;
}

}  // namespace dc

extern "C" int32_t dc_gemm_pair_slots(void) {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] { err = dc::preload_gemm_kernels(); });
  return err == cudaSuccess ? dc::pair_slots(0) : -1;
}

extern "C" uint64_t dc_gemm_workspace_bytes(void) { return dc::gemm_workspace_bytes(); }

extern "C" dc_status dc_gemm(const dc_gemm_args* g, cudaStream_t stream) {
  std::string err;
  dc_status s = dc::launch_gemm(g, stream, &err);
  if (s != DC_OK) dc::set_global_error(err);
  return s;
}

namespace dc {
cudaError_t preload_gemm_kernels() {
  cudaFuncAttributes a;
  cudaError_t e = cudaSuccess;
#define DC_ONE_ATTR(EPI_)                                                                          \
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, gemm_bf16_sm100<EPI_>);                      \
  if (e == cudaSuccess)                                                                            \
    e = cudaFuncSetAttribute(gemm_bf16_sm100<EPI_>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM);
  DC_ONE_ATTR(0)
  DC_ONE_ATTR(1)
#undef DC_ONE_ATTR
#define DC_PAIR_ATTR(BN_, ST_, EPI_)                                                               \
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, gemm2_bf16_sm100<BN_, ST_, EPI_>);           \
  if (e == cudaSuccess)                                                                            \
    e = cudaFuncSetAttribute(gemm2_bf16_sm100<BN_, ST_, EPI_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             Pair<BN_, ST_>::SMEM);
  DC_PAIR_ATTR(256, 7, 0)
  DC_PAIR_ATTR(256, 7, 1)
  DC_PAIR_ATTR(256, 6, 0)
  DC_PAIR_ATTR(256, 6, 1)
  DC_PAIR_ATTR(256, 6, 2)
  DC_PAIR_ATTR(256, 6, 3)
  DC_PAIR_ATTR(128, 9, 0)
  DC_PAIR_ATTR(128, 9, 1)
#undef DC_PAIR_ATTR
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(gemm2_bf16_sm100<256, 6, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Pair<256, 6>::SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(gemm2_bf16_sm100<256, 6, 0, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Pair<256, 6>::SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(gemm2_bf16_sm100<256, 7, 0, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Pair<256, 7>::SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(gemm2_bf16_sm100<256, 6, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Pair<256, 6>::SMEM);
  if (e == cudaSuccess) e = query_pair_slots<256, 6>(&g_pair_slots[0]);
  if (e == cudaSuccess) e = query_pair_slots<128, 9>(&g_pair_slots[1]);
  if (e == cudaSuccess) e = query_pair_slots<256, 7>(&g_pair_slots[2]);
  return e;
}
}  // namespace dc
