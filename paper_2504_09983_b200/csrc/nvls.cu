// NVLink SHARP (NVLS) forms of the two collectives, for an
// NVSwitch box where the symmetric buffers also have a multicast mapping
// (torch symmetric memory's multicast_ptr; dc_bind_multicast):
//
//  ag_multimem  (P:236 all-gather): every rank stores its shard of each member
//               ONCE, with 16-byte multimem.st to the multicast address of the
//               arena slot; the switch replicates the store into all N arenas.
//               A sender's NVLink egress is S_i bytes instead of (N-1) S_i.
//               Completion: one multimem.red.release of the done counter's
//               multicast address bumps it on every rank.  Same ready / done
//               protocol and targets as ag_push; bit-identical buffers.
//  rs_adam_nvls (P:127 / P:440 / P:504): owner r reads slice r of every rank's
//               bf16 grad with one multimem.ld_reduce (add, fp32 accumulate in
//               the switch, bf16 result) per 8 elements, then 1/N and the Adam
//               step of rs_adam.  NOT bit-exact with the ascending-rank fp32
//               sum (the switch fixes its own order and rounds the sum to
//               bf16): opt-in, checked within the north star's bf16 tolerance.
//
// Both need a multicast object, which the driver refuses on a one-GPU box
// (profiles/r01g/nvls/probe.txt); the executor uses them only when
// dc_bind_multicast gave non-zero addresses and option "nvls" asks for them.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "adam.cuh"
#include "dc_internal.h"
#include "ptx.cuh"

namespace dc {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ void multimem_st16(void* mc, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};"
               :: "l"(mc), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void multimem_red_add_release(uint32_t* mc, uint32_t v) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" :: "l"(mc), "r"(v) : "memory");
}
// 8 bf16 sums over the ranks of the multicast group (fp32 accumulation)
__device__ __forceinline__ uint4 multimem_ld_reduce_bf16x8(const void* mc) {
  uint4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(mc) : "memory");
  return r;
}

constexpr int AGM_MAXM = 48, AGM_THREADS = 256, AGM_UNR = 8;
struct AgMcParams {
  int nm;
  const uint4* src[AGM_MAXM];
  int64_t dst_off[AGM_MAXM];   // byte offset of this rank's slot in the arena
  int64_t nvec[AGM_MAXM];
  uint8_t* arena_mc;           // multicast address of the arena
  uint32_t* done_mc;           // multicast address of done[gid]
};

__global__ void __launch_bounds__(AGM_THREADS) ag_multimem_kernel(const AgMcParams p) {
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int mi = 0; mi < p.nm; ++mi) {
    const uint4* src = p.src[mi];
    uint4* dst = reinterpret_cast<uint4*>(p.arena_mc + p.dst_off[mi]);
    const int64_t n = p.nvec[mi];
    int64_t i = tid;
    for (; i + (AGM_UNR - 1) * nthr < n; i += AGM_UNR * nthr) {
      uint4 v[AGM_UNR];
#pragma unroll
      for (int u = 0; u < AGM_UNR; ++u) v[u] = __ldg(src + i + u * nthr);
#pragma unroll
      for (int u = 0; u < AGM_UNR; ++u) multimem_st16(dst + i + u * nthr, v[u]);
    }
    for (; i < n; i += nthr) multimem_st16(dst + i, __ldg(src + i));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    multimem_red_add_release(p.done_mc, 1u);     // done[gid] += 1 on every rank
  }
}

dc_status k_ag_multimem(const std::vector<AgMember>& mem, uint8_t* arena_mc, uint32_t* done_mc, int ctas,
                        const uint32_t* ready_local, int world, uint32_t epoch, const uint32_t* done_local,
                        uint32_t done_target, uint64_t timeout_ns, uint32_t* err_flag, cudaStream_t st,
                        cudaEvent_t ev_after_ready) {
  k_wait_flags(ready_local, world, epoch, timeout_ns, err_flag, st);
  if (ev_after_ready) record_event(ev_after_ready, st);
  for (size_t b = 0; b < mem.size(); b += AGM_MAXM) {
    AgMcParams p{};
    p.nm = (int)std::min<size_t>(AGM_MAXM, mem.size() - b);
    for (int i = 0; i < p.nm; ++i) {
      p.src[i] = reinterpret_cast<const uint4*>(mem[b + i].src);
      p.dst_off[i] = mem[b + i].dst_off_bytes;
      p.nvec[i] = mem[b + i].bytes / 16;
    }
    p.arena_mc = arena_mc;
    p.done_mc = done_mc;
    ag_multimem_kernel<<<ctas, AGM_THREADS, 0, st>>>(p);
    if (cudaGetLastError() != cudaSuccess) return DC_ECUDA;
    count_launch();
  }
  k_wait_flags(done_local, 1, done_target, timeout_ns, err_flag, st);
  return cudaGetLastError() == cudaSuccess ? DC_OK : DC_ECUDA;
}

// ------------------------------------------------------------------ rs_adam_nvls
constexpr int RSN_MAXM = 48, RSN_THREADS = 256;
struct RsMcParams {
  int nm, rank;
  int64_t goff[RSN_MAXM], S[RSN_MAXM], store_off[RSN_MAXM];
  const uint8_t* slot_mc;      // multicast address of this layer's grad slot
  uint32_t* consumed[MAXW];
  int world;
  uint32_t consumed_value;
  uint32_t* done_ctr;
  uint32_t done_target;
  float *master, *m, *v, *acc;
  bf16* shard;
  float w1, w2, b2, neg_s, c, eps, invN;
  const float* scal;
};

template <int MODE>
__global__ void __launch_bounds__(RSN_THREADS) rs_adam_nvls_kernel(const RsMcParams p) {
  const uint64_t pol = policy_evict_first();
  const AdamScalars a = adam_scalars(p.w1, p.w2, p.b2, p.scal ? -p.scal[0] : p.neg_s, p.scal ? p.scal[1] : p.c, p.eps, p.invN);
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int mi = 0; mi < p.nm; ++mi) {
    const int64_t n8 = p.S[mi] / 8;
    const uint8_t* gsl = p.slot_mc + p.goff[mi] + (int64_t)p.rank * p.S[mi] * 2;
    const int64_t so = p.store_off[mi];
    for (int64_t i = tid; i < n8; i += nthr) {
      const uint4 gs = multimem_ld_reduce_bf16x8(gsl + i * 16);
      if constexpr (MODE == RS_FIRST || MODE == RS_ADD) {
        float g[8];
        bf16x8_to_f32(gs, g);
        if constexpr (MODE == RS_ADD) {
          const uint4 a0 = ld_stream(p.acc + so + 8 * i, pol), a1 = ld_stream(p.acc + so + 8 * i + 4, pol);
          const float* f0 = reinterpret_cast<const float*>(&a0);
          const float* f1 = reinterpret_cast<const float*>(&a1);
#pragma unroll
          for (int j = 0; j < 4; ++j) { g[j] = __fadd_rn(f0[j], g[j]); g[4 + j] = __fadd_rn(f1[j], g[4 + j]); }
        }
        st_stream(p.acc + so + 8 * i, *reinterpret_cast<const uint4*>(&g[0]), pol);
        st_stream(p.acc + so + 8 * i + 4, *reinterpret_cast<const uint4*>(&g[4]), pol);
      } else {
        constexpr bool ACC = MODE == RS_FINAL;
        Group8<1> x;
        load_group8<1, ACC>(x, nullptr, 0, p.master + so + 8 * i, p.m + so + 8 * i, p.v + so + 8 * i, pol,
                            p.acc + so + 8 * i);
        x.G[0] = gs;                          // the switch's sum: one "rank" (+0.0 + sum = sum)
        finish_group8<1, ACC>(x, 1, p.master + so + 8 * i, p.m + so + 8 * i, p.v + so + 8 * i,
                              p.shard + so + 8 * i, a, pol);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t prev = atomicAdd(p.done_ctr, 1u);
    if (prev + 1 == p.done_target) {            // last CTA: every slice pulled
      __threadfence_system();
      for (int q = 0; q < p.world; ++q) ptx::st_release_sys(p.consumed[q], p.consumed_value);
    }
  }
}

dc_status k_rs_adam_nvls(const std::vector<RsMember>& mem, int world, int rank, const uint8_t* slot_mc,
                         const uint32_t* ready_local, uint32_t ready_target, PeerFlags consumed_peers,
                         uint32_t consumed_value, uint32_t* done_ctr, uint32_t done_target, float* master, float* m,
                         float* v, void* shard, float* acc, int mode, int micro_steps, float s, float c, double beta1,
                         double beta2, double eps, int ctas, uint64_t timeout_ns, uint32_t* err_flag, cudaStream_t st,
                         const float* dev_scalars) {
  if (mode < RS_UPDATE || mode > RS_FINAL || (mode != RS_UPDATE && !acc) || micro_steps < 1) return DC_EINVAL;
  if (mem.size() > (size_t)RSN_MAXM || !slot_mc) return DC_EINVAL;
  RsMcParams p{};
  p.nm = (int)mem.size();
  p.rank = rank;
  p.world = world;
  for (int i = 0; i < p.nm; ++i) {
    p.goff[i] = mem[i].goff_bytes;
    p.S[i] = mem[i].S;
    p.store_off[i] = mem[i].store_off;
  }
  p.slot_mc = slot_mc;
  for (int q = 0; q < world; ++q) p.consumed[q] = consumed_peers.p[q];
  p.consumed_value = consumed_value;
  p.done_ctr = done_ctr; p.done_target = done_target;
  p.master = master; p.m = m; p.v = v; p.acc = acc; p.shard = reinterpret_cast<bf16*>(shard);
  p.w1 = (float)(1.0 - beta1);
  p.w2 = (float)(1.0 - beta2);
  p.b2 = (float)beta2;
  p.neg_s = -s;
  p.c = c;
  p.eps = (float)eps;
  p.invN = (float)(1.0 / ((double)world * micro_steps));
  p.scal = dev_scalars;
  k_wait_flags(ready_local, world, ready_target, timeout_ns, err_flag, st);
  switch (mode) {
    case RS_UPDATE: rs_adam_nvls_kernel<RS_UPDATE><<<ctas, RSN_THREADS, 0, st>>>(p); break;
    case RS_FIRST: rs_adam_nvls_kernel<RS_FIRST><<<ctas, RSN_THREADS, 0, st>>>(p); break;
    case RS_ADD: rs_adam_nvls_kernel<RS_ADD><<<ctas, RSN_THREADS, 0, st>>>(p); break;
    default: rs_adam_nvls_kernel<RS_FINAL><<<ctas, RSN_THREADS, 0, st>>>(p); break;
  }
  if (cudaGetLastError() != cudaSuccess) return DC_ECUDA;
  count_launch();
  return DC_OK;
}

cudaError_t preload_nvls_kernels() {
  cudaFuncAttributes a;
  const void* fns[] = {(const void*)ag_multimem_kernel, (const void*)rs_adam_nvls_kernel<RS_UPDATE>,
                       (const void*)rs_adam_nvls_kernel<RS_FIRST>, (const void*)rs_adam_nvls_kernel<RS_ADD>,
                       (const void*)rs_adam_nvls_kernel<RS_FINAL>};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace dc
