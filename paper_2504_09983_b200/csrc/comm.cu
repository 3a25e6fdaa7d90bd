// Collective kernels of the sharded-parameter life cycle, over peer-mapped
// memory (NVLink 5 / NVSwitch at N > 1; plain device memory of the other
// virtual ranks in DC_VIRTUAL_RANKS mode).
//
//  ag_push  (P:236 all-gather): every rank stores its shard of each member of a
//           gather group into every rank's arena with 16-byte st.global —
//           one local HBM read, N peer writes per vector.  Write-after-read on
//           the receivers' arena is guarded by ready flags (posted by the
//           receiver's release of the previous occupant); completion by
//           per-gather done counters bumped with red.release.sys.
//  rs_adam  (reduce-scatter + 1/N + Adam, P:127 / P:440 / P:504): owner r pulls
//           slice r of every rank's bf16 grad slot (peer loads), sums in fp32
//           in ascending rank order from +0.0, scales by 1/N and applies the
//           Adam step to its fp32 master/m/v shard, writing the bf16 shard.
//
// Flag waits are bounded (globaltimer); a timeout sets a host-mapped error word
// instead of hanging the GPU.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "adam.cuh"
#include "dc_internal.h"
#include "ptx.cuh"

namespace dc {

using bf16 = __nv_bfloat16;

constexpr int AG_MAXM = 48;
struct AgParams {
  int nm, world, rank;
  const uint4* src[AG_MAXM];
  int64_t dst_off[AG_MAXM];   // byte offset of this rank's slot inside each arena
  int64_t nvec[AG_MAXM];      // 16-byte vectors of the member's shard
  uint8_t* arena[MAXW];
  uint32_t* done_peer[MAXW];  // &done[gid] in every rank's flag table
  const uint32_t* ready;      // &ready[gid * world] in this rank's table
  const uint32_t* done_local;
  uint32_t epoch, done_target;
  int wait;
  uint64_t timeout_ns;
  uint32_t* err;
};

// "counter >= target" in serial-number arithmetic: the gather done counters
// grow without reset in eager mode, so a plain `<` would see a stale counter
// as already past a target that wrapped around 2^32
__device__ __forceinline__ bool spin_ge(const uint32_t* p, uint32_t target, uint64_t t0, uint64_t tmo,
                                        uint32_t* err, uint32_t code) {
  uint32_t seen;
  while ((int32_t)((seen = ptx::ld_acquire_sys(p)) - target) < 0) {
    if (ptx::globaltimer() - t0 > tmo) {
      if (atomicCAS(err + 1, 0u, 1u) == 0u) {      // claim the record
        err[2] = target;
        err[3] = seen;
        err[4] = (uint32_t)reinterpret_cast<uintptr_t>(p);
        err[5] = (uint32_t)(reinterpret_cast<uintptr_t>(p) >> 32);
        __threadfence_system();
        atomicExch(err, code);                      // published last: the host reads code first
      }
      return false;
    }
    __nanosleep(64);
  }
  return true;
}

// Flag waits run in separate one-thread kernels on the same stream (before the
// push: every receiver's ready flag; after it: this rank's done counter), so a
// waiting rank occupies one SM slot, never a whole grid of spinning CTAs.
// 256 threads x <= 64 registers: a push CTA fits beside a CTA of the pair GEMM
// (384 threads x 120 registers) on one SM (65536 registers), so a prefetched
// gather really runs during the layer GEMMs; 8 x 16 B stores in flight per
// thread keep ~2 MB outstanding at 64 CTAs (NVLink latency x 900 GB/s).
constexpr int AG_THREADS = 256, AG_UNR = 8;
__global__ void __launch_bounds__(AG_THREADS) ag_push_kernel(const AgParams p) {
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int m = 0; m < p.nm; ++m) {
    const uint4* src = p.src[m];
    const int64_t n = p.nvec[m];
    const int64_t off = p.dst_off[m];
    int64_t i = tid;
    for (; i + (AG_UNR - 1) * nthr < n; i += AG_UNR * nthr) {
      uint4 v[AG_UNR];
#pragma unroll
      for (int u = 0; u < AG_UNR; ++u) v[u] = __ldg(src + i + u * nthr);
      // destinations rotated by rank: the N senders start on N different
      // receivers instead of all on rank 0 (spreads NVSwitch ingress)
      for (int qq = 0; qq < p.world; ++qq) {
        const int q = (qq + p.rank) % p.world;
        uint4* dst = reinterpret_cast<uint4*>(p.arena[q] + off);
#pragma unroll
        for (int u = 0; u < AG_UNR; ++u) dst[i + u * nthr] = v[u];
      }
    }
    for (; i < n; i += nthr) {
      const uint4 v = __ldg(src + i);
      for (int qq = 0; qq < p.world; ++qq) reinterpret_cast<uint4*>(p.arena[(qq + p.rank) % p.world] + off)[i] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < p.world; ++q) ptx::red_add_release_sys(p.done_peer[q], 1u);
  }
}

// Chunked push (fused all-gather -> GEMM): the same stores as
// ag_push, but chunk by chunk (chunk j of member m = elements
// [j E, min((j+1) E, S)) of this rank's shard; CTA b takes chunks b, b + grid,
// ... of the members' chunk list in order, so the first chunks land first),
// and after each chunk's stores have landed on every receiver the CTA writes
// the gather's value into chunk[param][rank][j] of every receiver's flag
// table: a GEMM there may start on the rows that already arrived.
struct AgChunkParams {
  int nm, world, rank;
  const uint4* src[AG_MAXM];
  int64_t dst_off[AG_MAXM];
  int64_t nvec[AG_MAXM];
  int64_t evec[AG_MAXM];      // 16-byte vectors per chunk
  int cum[AG_MAXM + 1];       // chunk list prefix: member m owns chunks [cum[m], cum[m + 1])
  int64_t word[AG_MAXM];      // chunk[param][rank][0] word in every table
  uint32_t value[AG_MAXM];
  uint8_t* arena[MAXW];
  uint32_t* flags[MAXW];      // every rank's flag table
  uint32_t* done_peer[MAXW];
};

__global__ void __launch_bounds__(AG_THREADS) ag_push_chunked_kernel(const AgChunkParams p) {
  int m = 0;
  for (int c = blockIdx.x; c < p.cum[p.nm]; c += gridDim.x) {
    while (c >= p.cum[m + 1]) ++m;
    const int j = c - p.cum[m];
    const int64_t v0 = (int64_t)j * p.evec[m];
    const int64_t v1 = min(v0 + p.evec[m], p.nvec[m]);
    const uint4* src = p.src[m];
    for (int64_t i = v0 + threadIdx.x; i < v1; i += AG_UNR * AG_THREADS) {
      uint4 v[AG_UNR];
#pragma unroll
      for (int u = 0; u < AG_UNR; ++u)
        if (i + u * AG_THREADS < v1) v[u] = __ldg(src + i + u * AG_THREADS);
      for (int qq = 0; qq < p.world; ++qq) {
        uint4* dst = reinterpret_cast<uint4*>(p.arena[(qq + p.rank) % p.world] + p.dst_off[m]);
#pragma unroll
        for (int u = 0; u < AG_UNR; ++u)
          if (i + u * AG_THREADS < v1) dst[i + u * AG_THREADS] = v[u];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int q = 0; q < p.world; ++q) ptx::st_release_sys(p.flags[q] + p.word[m] + j, p.value[m]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < p.world; ++q) ptx::red_add_release_sys(p.done_peer[q], 1u);
  }
}

// testing (option ag_delay_us): hold the AG stream so the consumers start first
__global__ void delay_kernel(uint32_t us) {
  const uint64_t t0 = ptx::globaltimer();
  while (ptx::globaltimer() - t0 < (uint64_t)us * 1000u) __nanosleep(1000);
}

__global__ void wait_flags_kernel(const uint32_t* f, int n, uint32_t target, uint64_t tmo, uint32_t* err,
                                  uint32_t code) {
  const uint64_t t0 = ptx::globaltimer();
  for (int i = 0; i < n; ++i)
    if (!spin_ge(f + i, target, t0, tmo, err, code | i)) return;
}

dc_status launch_ag_bulk(const std::vector<AgMember>& mem, int world, int rank, const uint64_t* arena_peers,
                         PeerFlags done_peers, int ctas, cudaStream_t st);

dc_status k_ag_push(const std::vector<AgMember>& mem, int world, int rank, const uint64_t* arena_peers,
                    const uint32_t* ready_local, uint32_t epoch, PeerFlags done_peers, const uint32_t* done_local,
                    uint32_t done_target, int ctas, uint64_t timeout_ns, uint32_t* err_flag, cudaStream_t st,
                    cudaEvent_t ev_after_ready, bool skip_waits, uint32_t delay_us, const uint64_t* flag_peers,
                    bool bulk) {
  if (!skip_waits) {
    wait_flags_kernel<<<1, 1, 0, st>>>(ready_local, world, epoch, timeout_ns, err_flag, 0x100u);
    count_launch();
  }
  if (ev_after_ready) record_event(ev_after_ready, st);
  if (delay_us) {
    delay_kernel<<<1, 1, 0, st>>>(delay_us);
    count_launch();
  }
  if (bulk && (mem.empty() || mem[0].chunk_word < 0)) {   // bulk-copy pipeline (option ag_bulk)
    dc_status r = launch_ag_bulk(mem, world, rank, arena_peers, done_peers, ctas, st);
    if (r != DC_OK) return r;
    if (!skip_waits) {
      wait_flags_kernel<<<1, 1, 0, st>>>(done_local, 1, done_target, timeout_ns, err_flag, 0x200u);
      count_launch();
    }
    return cudaGetLastError() == cudaSuccess ? DC_OK : DC_ECUDA;
  }
  if (!mem.empty() && mem[0].chunk_word >= 0) {   // chunked pushes (fused all-gather -> GEMM)
    if (!flag_peers) return DC_EINVAL;
    for (size_t b = 0; b < mem.size(); b += AG_MAXM) {
      AgChunkParams p{};
      p.nm = (int)std::min<size_t>(AG_MAXM, mem.size() - b);
      p.world = world; p.rank = rank;
      p.cum[0] = 0;
      for (int i = 0; i < p.nm; ++i) {
        const AgMember& a = mem[b + i];
        p.src[i] = reinterpret_cast<const uint4*>(a.src);
        p.dst_off[i] = a.dst_off_bytes;
        p.nvec[i] = a.bytes / 16;
        p.evec[i] = ag_chunk_elems(a.bytes / 2) / 8;
        p.cum[i + 1] = p.cum[i] + (int)((p.nvec[i] + p.evec[i] - 1) / p.evec[i]);
        p.word[i] = a.chunk_word;
        p.value[i] = a.chunk_value;
      }
      for (int q = 0; q < world; ++q) {
        p.arena[q] = reinterpret_cast<uint8_t*>(arena_peers[q]);
        p.flags[q] = reinterpret_cast<uint32_t*>(flag_peers[q]);
        p.done_peer[q] = done_peers.p[q];
      }
      ag_push_chunked_kernel<<<ctas, AG_THREADS, 0, st>>>(p);
      if (cudaGetLastError() != cudaSuccess) return DC_ECUDA;
      count_launch();
    }
    if (!skip_waits) {
      wait_flags_kernel<<<1, 1, 0, st>>>(done_local, 1, done_target, timeout_ns, err_flag, 0x200u);
      count_launch();
    }
    return cudaGetLastError() == cudaSuccess ? DC_OK : DC_ECUDA;
  }
  // members beyond AG_MAXM go to extra launches
  for (size_t b = 0; b < mem.size(); b += AG_MAXM) {
    AgParams p{};
    p.nm = (int)std::min<size_t>(AG_MAXM, mem.size() - b);
    p.world = world; p.rank = rank;
    for (int i = 0; i < p.nm; ++i) {
      const AgMember& a = mem[b + i];
      p.src[i] = reinterpret_cast<const uint4*>(a.src);
      p.dst_off[i] = a.dst_off_bytes;
      p.nvec[i] = a.bytes / 16;
    }
    for (int q = 0; q < world; ++q) {
      p.arena[q] = reinterpret_cast<uint8_t*>(arena_peers[q]);
      p.done_peer[q] = done_peers.p[q];
    }
    p.ready = ready_local;
    p.done_local = done_local;
    p.epoch = epoch;
    p.done_target = done_target;
    p.wait = (b + AG_MAXM >= mem.size());
    p.timeout_ns = timeout_ns;
    p.err = err_flag;
    ag_push_kernel<<<ctas, AG_THREADS, 0, st>>>(p);
    if (cudaGetLastError() != cudaSuccess) return DC_ECUDA;
    count_launch();
  }
  if (!skip_waits) {
    wait_flags_kernel<<<1, 1, 0, st>>>(done_local, 1, done_target, timeout_ns, err_flag, 0x200u);
    count_launch();
  }
  return cudaGetLastError() == cudaSuccess ? DC_OK : DC_ECUDA;
}

// ------------------------------------------------------------------ rs_adam
constexpr int RS_MAXM = 48;
struct RsParams {
  int nm, world, rank;
  int64_t goff[RS_MAXM];      // byte offset of member's padded tensor in a grad slot
  int64_t S[RS_MAXM];
  int64_t store_off[RS_MAXM];
  const uint8_t* slot[MAXW];  // this layer's grad slot on every rank
  const uint32_t* ready;      // grad-ready flags [world] in this rank's table
  uint32_t ready_target;
  uint32_t* consumed[MAXW];   // consumed[slot][rank] in every rank's table
  uint32_t consumed_value;
  uint32_t* done_ctr;
  uint32_t done_target;
  float* master; float* m; float* v; bf16* shard;
  float* acc;                 // fp32 accumulated grad shard (gradient accumulation)
  float w1, w2, b2, neg_s, c, eps, invN;
  const float* scal;          // graph mode: (s, c) of the step in device memory, else null
  uint64_t timeout_ns;
  uint32_t* err;
};

#ifndef DC_RS_UNR
#define DC_RS_UNR 2           // N > 1: two groups' peer loads in flight per thread (NVLink latency)
#endif
#ifndef DC_RS_UNR_N1
#define DC_RS_UNR_N1 1        // N = 1: one group (80 registers; 12-15 % faster in-step than two groups
#endif                        // at 112 registers, profiles/r01g/rs_coresidency_ab.md)
// groups of 8 elements per thread per iteration (loads hoisted)
// (the accumulate-only modes keep two: few registers, few bytes per element)
template <int MAXQ, int MODE>
struct RsUnr {
  static constexpr int value = (MAXQ == 1 && (MODE == RS_UPDATE || MODE == RS_FINAL)) ? DC_RS_UNR_N1 : DC_RS_UNR;
};

// MODE (gradient accumulation; dc.h dc_reduce_scatter_step):
//   RS_UPDATE  g = sum * 1/N, Adam                      (n = 1)
//   RS_FIRST   acc = sum                                (micro-step 0 of n > 1)
//   RS_ADD     acc = acc + sum                          (micro-steps 1 .. n-2)
//   RS_FINAL   g = (acc + sum) * 1/(N n), Adam          (micro-step n-1)
#ifndef DC_RS_MINB
#define DC_RS_MINB 1          // min resident CTAs per SM for the register budget (A/B)
#endif
template <int MAXQ, int MODE>
__global__ void __launch_bounds__(256, DC_RS_MINB) rs_adam_kernel(const RsParams p) {
  constexpr int RS_UNR = RsUnr<MAXQ, MODE>::value;
  {   // grad-ready of every rank was awaited by the preceding wait kernel
    const uint64_t pol = policy_evict_first();
    const AdamScalars a = adam_scalars(p.w1, p.w2, p.b2, p.scal ? -p.scal[0] : p.neg_s, p.scal ? p.scal[1] : p.c, p.eps, p.invN);
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int mi = 0; mi < p.nm; ++mi) {
      const int64_t n8 = p.S[mi] / 8;
      const int64_t gbase = p.goff[mi] + (int64_t)p.rank * p.S[mi] * 2;
      float* mst = p.master + p.store_off[mi];
      float* mm = p.m + p.store_off[mi];
      float* vv = p.v + p.store_off[mi];
      float* acc = p.acc + p.store_off[mi];
      bf16* sh = p.shard + p.store_off[mi];
      if constexpr (MODE == RS_FIRST || MODE == RS_ADD) {
        for (int64_t i0 = tid; i0 < n8; i0 += nthr * RS_UNR) {
          uint4 G[RS_UNR][MAXQ], A[RS_UNR][2];
#pragma unroll
          for (int u = 0; u < RS_UNR; ++u) {
            const int64_t i = i0 + u * nthr;
            if (i < n8) {
#pragma unroll
              for (int q = 0; q < MAXQ; ++q)
                if (q < p.world) G[u][q] = ld_stream(p.slot[q] + gbase + i * 16, pol);
              if constexpr (MODE == RS_ADD) {
                A[u][0] = ld_stream(acc + 8 * i, pol);
                A[u][1] = ld_stream(acc + 8 * i + 4, pol);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < RS_UNR; ++u) {
            const int64_t i = i0 + u * nthr;
            if (i < n8) {
              float g[8];
              sum_ranks8<MAXQ>(G[u], p.world, g);
              if constexpr (MODE == RS_ADD) {
                const float* af = reinterpret_cast<const float*>(&A[u][0]);
#pragma unroll
                for (int j = 0; j < 8; ++j) g[j] = __fadd_rn(af[j], g[j]);
              }
              st_stream(acc + 8 * i, *reinterpret_cast<const uint4*>(&g[0]), pol);
              st_stream(acc + 8 * i + 4, *reinterpret_cast<const uint4*>(&g[4]), pol);
            }
          }
        }
      } else {
        constexpr bool ACC = MODE == RS_FINAL;
        for (int64_t i0 = tid; i0 < n8; i0 += nthr * RS_UNR) {
          Group8<MAXQ> x[RS_UNR];
#pragma unroll
          for (int u = 0; u < RS_UNR; ++u) {     // every load of RS_UNR groups before any math
            const int64_t i = i0 + u * nthr;
            if (i < n8) {
              const uint8_t* gp[MAXQ];
#pragma unroll
              for (int q = 0; q < MAXQ; ++q) gp[q] = q < p.world ? p.slot[q] + gbase + i * 16 : nullptr;
              load_group8<MAXQ, ACC>(x[u], gp, p.world, mst + 8 * i, mm + 8 * i, vv + 8 * i, pol, acc + 8 * i);
            }
          }
#pragma unroll
          for (int u = 0; u < RS_UNR; ++u) {
            const int64_t i = i0 + u * nthr;
            if (i < n8)
              finish_group8<MAXQ, ACC>(x[u], p.world, mst + 8 * i, mm + 8 * i, vv + 8 * i, sh + 8 * i, a, pol);
          }
        }
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

// ------------------------------------------------------------------ rs_adam (bulk-copy pipeline)
// The same arithmetic as rs_adam_kernel (UPDATE / FINAL modes), with the
// memory side moved onto the copy engines of the SM: one producer thread
// streams 2048-element chunks of every input (fp32 master / m / v [/ acc], the
// bf16 grad slice of every rank) into a ring of shared-memory stages with
// cp.async.bulk (completion on an mbarrier), 16 consumer warps apply the
// update in place in shared memory (4 elements per thread: conflict-free
// 16-byte accesses) and one consumer thread writes the stage back with bulk
// stores.  The loads of the next stages stay in flight while the consumers do
// the IEEE divisions / square roots, so the HBM stream does not stall on the
// arithmetic (the register-bound LDG kernel keeps ~2 groups of 8 elements in
// flight per thread and alternates between the two).
constexpr int RSB_CH = RS_BULK_CHUNK;        // elements per chunk
constexpr int RSB_CONSUMERS = 512;           // 16 warps, 4 elements each per chunk
constexpr int RSB_THREADS = RSB_CONSUMERS + 32;
#ifndef DC_RSB_CTAS_PER_SM
#define DC_RSB_CTAS_PER_SM 2    // two independent pipelines per SM: one CTA's arithmetic overlaps the other's barrier / store turn
#endif
constexpr int RSB_CTAS_PER_SM = DC_RSB_CTAS_PER_SM;
int rs_bulk_ctas_per_sm() { return RSB_CTAS_PER_SM; }

template <int MAXQ, bool ACC>
struct RsBulk {
  static constexpr int STAGE = RSB_CH * (12 + 2 * MAXQ + 2 + (ACC ? 4 : 0));   // p m v, grads, shard, acc
  static constexpr int BUDGET = (220 * 1024) / RSB_CTAS_PER_SM;
  static constexpr int ST0 = BUDGET / STAGE < 8 ? BUDGET / STAGE : 8;
  static constexpr int ST = ST0 < 2 ? 2 : ST0;
  static constexpr int SMEM = ST * STAGE + 2 * ST * 8 + 128;
};

__device__ __forceinline__ void bulk_g2s(void* s, const void* g, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               :: "r"(ptx::smem_u32(s)), "l"(g), "r"(bytes), "r"(ptx::smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* s, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
               :: "l"(g), "r"(ptx::smem_u32(s)), "r"(bytes), "l"(pol) : "memory");
}

// ------------------------------------------------------------------ ag_push (bulk-copy pipeline)
// The push with its data path on the SM's bulk-copy (TMA) engine instead of
// per-thread 16-byte loads / stores: one thread streams PIECE-byte pieces of
// the members' shards into a ring of AGB_ST shared-memory stages
// (cp.async.bulk global -> shared, mbarrier completion) and, for each landed
// piece, issues one bulk store per receiver (cp.async.bulk shared -> global,
// bulk groups; ranks rotated as in ag_push).  A stage is refilled once its
// stores have READ it (wait_group.read), so the next pieces' loads stay in
// flight behind the stores.  32 KB of shared memory and one warp per CTA: it
// fits beside a pair-GEMM CTA (193 KB, 384 threads).  Completion: wait_group 0
// (stores performed), proxy fence, system fence, red.release.sys of every
// receiver's done counter — the same done protocol as ag_push.
constexpr int AGB_PIECE = 8192, AGB_ST = 4, AGB_SMEM = AGB_PIECE * AGB_ST + 128;
struct AgBulkParams {
  int nm, world, rank;
  const uint8_t* src[AG_MAXM];
  int64_t dst_off[AG_MAXM];
  int64_t bytes[AG_MAXM];
  int cum[AG_MAXM + 1];       // piece list prefix: member m owns pieces [cum[m], cum[m + 1])
  uint8_t* arena[MAXW];
  uint32_t* done_peer[MAXW];
};

__global__ void __launch_bounds__(32) ag_push_bulk_kernel(const AgBulkParams p) {
  extern __shared__ __align__(128) uint8_t agb_smem[];
  uint8_t* buf = agb_smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(agb_smem + AGB_PIECE * AGB_ST);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < AGB_ST; ++s) ptx::mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t pol = policy_evict_first();
  const int total = p.cum[p.nm];
  // piece k of this CTA = global piece blockIdx.x + k * gridDim.x
  auto locate = [&](int c, int& m, int64_t& off, uint32_t& n) {
    m = 0;
    while (c >= p.cum[m + 1]) ++m;
    off = (int64_t)(c - p.cum[m]) * AGB_PIECE;
    const int64_t rem = p.bytes[m] - off;
    n = (uint32_t)(rem < AGB_PIECE ? rem : AGB_PIECE);
  };
  auto load = [&](int k) {
    const int c = blockIdx.x + k * gridDim.x;
    if (c >= total) return;
    int m; int64_t off; uint32_t n;
    locate(c, m, off, n);
    uint64_t* bar = &full[k % AGB_ST];
    ptx::mbar_arrive_expect_tx(bar, n);
    bulk_g2s(buf + (k % AGB_ST) * AGB_PIECE, p.src[m] + off, n, bar, pol);
  };
  // loads run AGB_AHEAD pieces ahead; the stores of up to AGB_ST - AGB_AHEAD
  // pieces stay in flight (a stage is refilled once the stores of the piece
  // that used it AGB_ST pieces earlier have read it)
  constexpr int AGB_AHEAD = 2;
  for (int k = 0; k < AGB_AHEAD; ++k) load(k);
  for (int k = 0;; ++k) {
    const int c = blockIdx.x + k * gridDim.x;
    if (c >= total) break;
    int m; int64_t off; uint32_t n;
    locate(c, m, off, n);
    ptx::mbar_wait(&full[k % AGB_ST], (k / AGB_ST) & 1);
    const uint8_t* st = buf + (k % AGB_ST) * AGB_PIECE;
    for (int qq = 0; qq < p.world; ++qq) {
      uint8_t* dst = p.arena[(qq + p.rank) % p.world] + p.dst_off[m] + off;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   :: "l"(dst), "r"(ptx::smem_u32(st)), "r"(n) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // piece k + AHEAD goes to the stage of piece k + AHEAD - ST: its stores
    // (committed ST - AHEAD groups ago) must have read it
    asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(AGB_ST - AGB_AHEAD) : "memory");
    load(k + AGB_AHEAD);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");      // every store performed
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __threadfence_system();
  for (int q = 0; q < p.world; ++q) ptx::red_add_release_sys(p.done_peer[q], 1u);
}

dc_status launch_ag_bulk(const std::vector<AgMember>& mem, int world, int rank, const uint64_t* arena_peers,
                         PeerFlags done_peers, int ctas, cudaStream_t st) {
  for (size_t b = 0; b < mem.size(); b += AG_MAXM) {
    AgBulkParams p{};
    p.nm = (int)std::min<size_t>(AG_MAXM, mem.size() - b);
    p.world = world; p.rank = rank;
    p.cum[0] = 0;
    for (int i = 0; i < p.nm; ++i) {
      const AgMember& a = mem[b + i];
      p.src[i] = reinterpret_cast<const uint8_t*>(a.src);
      p.dst_off[i] = a.dst_off_bytes;
      p.bytes[i] = a.bytes;
      p.cum[i + 1] = p.cum[i] + (int)((a.bytes + AGB_PIECE - 1) / AGB_PIECE);
    }
    for (int q = 0; q < world; ++q) {
      p.arena[q] = reinterpret_cast<uint8_t*>(arena_peers[q]);
      p.done_peer[q] = done_peers.p[q];
    }
    ag_push_bulk_kernel<<<ctas, 32, AGB_SMEM, st>>>(p);
    if (cudaGetLastError() != cudaSuccess) return DC_ECUDA;
    count_launch();
  }
  return DC_OK;
}

template <int MAXQ, int MODE>
__global__ void __launch_bounds__(RSB_THREADS, RSB_CTAS_PER_SM) rs_adam_bulk_kernel(const RsParams p) {
  constexpr bool ACC = MODE == RS_FINAL;
  using B = RsBulk<MAXQ, ACC>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + B::ST * B::STAGE);
  uint64_t* empty = full + B::ST;
  // member chunk prefix (units = chunks of RSB_CH elements, member-major)
  __shared__ int64_t cum[RS_MAXM + 1];
  if (threadIdx.x == 0) {
    cum[0] = 0;
    for (int i = 0; i < p.nm; ++i) cum[i + 1] = cum[i] + (p.S[i] + RSB_CH - 1) / RSB_CH;
    for (int s = 0; s < B::ST; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int64_t units = cum[p.nm];
  const uint64_t pol = policy_evict_first();
  auto locate = [&](int64_t u, int& mi, int64_t& e0, int& n) {
    mi = 0;
    while (cum[mi + 1] <= u) ++mi;
    e0 = (u - cum[mi]) * RSB_CH;
    const int64_t rem = p.S[mi] - e0;
    n = (int)(rem < RSB_CH ? rem : RSB_CH);
  };
  const int warp = threadIdx.x / 32;
  if (warp == RSB_CONSUMERS / 32) {            // producer warp: one thread issues every load
    if (threadIdx.x % 32 == 0) {
      int k = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++k) {
        const int s = k % B::ST;
        if (k >= B::ST) ptx::mbar_wait(&empty[s], ((k / B::ST) - 1) & 1);
        int mi, n;
        int64_t e0;
        locate(u, mi, e0, n);
        uint8_t* b = smem + (size_t)s * B::STAGE;
        const int64_t so = p.store_off[mi] + e0;
        const uint32_t f4 = (uint32_t)n * 4, h2 = (uint32_t)n * 2;
        ptx::mbar_arrive_expect_tx(&full[s], 3 * f4 + p.world * h2 + (ACC ? f4 : 0));
        bulk_g2s(b, p.master + so, f4, &full[s], pol);
        bulk_g2s(b + RSB_CH * 4, p.m + so, f4, &full[s], pol);
        bulk_g2s(b + RSB_CH * 8, p.v + so, f4, &full[s], pol);
        const int64_t gb = p.goff[mi] + ((int64_t)p.rank * p.S[mi] + e0) * 2;
        for (int q = 0; q < p.world; ++q) bulk_g2s(b + RSB_CH * (12 + 2 * q), p.slot[q] + gb, h2, &full[s], pol);
        if constexpr (ACC) bulk_g2s(b + RSB_CH * (14 + 2 * MAXQ), p.acc + so, f4, &full[s], pol);
      }
    }
  } else {                                     // consumers
    const AdamScalars a = adam_scalars(p.w1, p.w2, p.b2, p.scal ? -p.scal[0] : p.neg_s, p.scal ? p.scal[1] : p.c, p.eps, p.invN);
    const int t = threadIdx.x;
    int k = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++k) {
      const int s = k % B::ST;
      int mi, n;
      int64_t e0;
      locate(u, mi, e0, n);
      ptx::mbar_wait(&full[s], (k / B::ST) & 1);
      uint8_t* b = smem + (size_t)s * B::STAGE;
      if (4 * t < n) {
        float4* P = reinterpret_cast<float4*>(b) + t;
        float4* M = reinterpret_cast<float4*>(b + RSB_CH * 4) + t;
        float4* V = reinterpret_cast<float4*>(b + RSB_CH * 8) + t;
        float g[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {       // ascending rank from +0.0 (reading D19)
          if (q < p.world) {
            const uint2 raw = reinterpret_cast<const uint2*>(b + RSB_CH * (12 + 2 * q))[t];
            const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
            const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
            g[0] = __fadd_rn(g[0], lo.x); g[1] = __fadd_rn(g[1], lo.y);
            g[2] = __fadd_rn(g[2], hi.x); g[3] = __fadd_rn(g[3], hi.y);
          }
        }
        if constexpr (ACC) {
          const float4 A = reinterpret_cast<const float4*>(b + RSB_CH * (14 + 2 * MAXQ))[t];
          g[0] = __fadd_rn(A.x, g[0]); g[1] = __fadd_rn(A.y, g[1]);
          g[2] = __fadd_rn(A.z, g[2]); g[3] = __fadd_rn(A.w, g[3]);
        }
        float4 pp = *P, mm = *M, vv = *V;
        constexpr bool kScale = !(MAXQ == 1 && MODE == RS_UPDATE);   // N = 1, n = 1: 1/N = 1 exactly
        adam_elem<kScale>(g[0], pp.x, mm.x, vv.x, a);
        adam_elem<kScale>(g[1], pp.y, mm.y, vv.y, a);
        adam_elem<kScale>(g[2], pp.z, mm.z, vv.z, a);
        adam_elem<kScale>(g[3], pp.w, mm.w, vv.w, a);
        *P = pp; *M = mm; *V = vv;
        const __nv_bfloat162 s0 = __floats2bfloat162_rn(pp.x, pp.y), s1 = __floats2bfloat162_rn(pp.z, pp.w);
        uint2 o;
        o.x = *reinterpret_cast<const uint32_t*>(&s0);
        o.y = *reinterpret_cast<const uint32_t*>(&s1);
        reinterpret_cast<uint2*>(b + RSB_CH * (12 + 2 * MAXQ))[t] = o;
      }
      ptx::fence_proxy_async_smem();           // generic-proxy smem writes -> visible to the bulk stores
      ptx::named_bar_sync(1, RSB_CONSUMERS);
      if (t == 0) {
        const int64_t so = p.store_off[mi] + e0;
        const uint32_t f4 = (uint32_t)n * 4;
        bulk_s2g(p.master + so, b, f4, pol);
        bulk_s2g(p.m + so, b + RSB_CH * 4, f4, pol);
        bulk_s2g(p.v + so, b + RSB_CH * 8, f4, pol);
        bulk_s2g(p.shard + so, b + RSB_CH * (12 + 2 * MAXQ), (uint32_t)n * 2, pol);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // every store group but the newest has finished reading its stage:
        // hand the previous stage back to the producer
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        if (k >= 1) ptx::mbar_arrive(&empty[(k - 1) % B::ST]);
      }
    }
    if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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

dc_status k_rs_adam(const std::vector<RsMember>& mem, int world, int rank, const uint64_t* slot_peers,
                    const uint32_t* ready_local, uint32_t ready_target, PeerFlags consumed_peers,
                    uint32_t consumed_value, uint32_t* done_ctr, uint32_t done_target, float* master, float* m,
                    float* v, void* shard, float* acc, int mode, int micro_steps, float s, float c, double beta1,
                    double beta2, double eps, int ctas, int threads, uint64_t timeout_ns, uint32_t* err_flag,
                    cudaStream_t st, const float* dev_scalars, bool bulk) {
  if (threads != 128 && threads != 256) return DC_EINVAL;
  if (mode < RS_UPDATE || mode > RS_FINAL || (mode != RS_UPDATE && !acc) || micro_steps < 1) return DC_EINVAL;
  if (mem.size() > (size_t)RS_MAXM) return DC_EINVAL;
  RsParams p{};
  p.nm = (int)mem.size();
  p.world = world; p.rank = rank;
  for (int i = 0; i < p.nm; ++i) {
    p.goff[i] = mem[i].goff_bytes;
    p.S[i] = mem[i].S;
    p.store_off[i] = mem[i].store_off;
  }
  for (int q = 0; q < world; ++q) {
    p.slot[q] = reinterpret_cast<const uint8_t*>(slot_peers[q]);
    p.consumed[q] = consumed_peers.p[q];
  }
  p.ready = ready_local; p.ready_target = ready_target;
  p.consumed_value = consumed_value;
  p.done_ctr = done_ctr; p.done_target = done_target;
  p.master = master; p.m = m; p.v = v; p.shard = reinterpret_cast<bf16*>(shard);
  p.acc = acc;
  p.w1 = (float)(1.0 - beta1);          // fp32(1 - b1) rounded once from double
  p.w2 = (float)(1.0 - beta2);
  p.b2 = (float)beta2;
  p.neg_s = -s;
  p.c = c;
  p.scal = dev_scalars;
  p.eps = (float)eps;
  p.invN = (float)(1.0 / ((double)world * micro_steps));   // fp32(1/(N n)), one rounding
  p.timeout_ns = timeout_ns;
  p.err = err_flag;
  wait_flags_kernel<<<1, 1, 0, st>>>(ready_local, world, ready_target, timeout_ns, err_flag, 0x300u);
  count_launch();
  auto launch = [&](auto mode_c) {
    constexpr int MODE = decltype(mode_c)::value;
    if (bulk && (MODE == RS_UPDATE || MODE == RS_FINAL)) {   // bulk-copy pipeline, one CTA per SM
      constexpr bool ACC = MODE == RS_FINAL;
      if (world == 1) rs_adam_bulk_kernel<1, MODE><<<ctas, RSB_THREADS, RsBulk<1, ACC>::SMEM, st>>>(p);
      else if (world == 2) rs_adam_bulk_kernel<2, MODE><<<ctas, RSB_THREADS, RsBulk<2, ACC>::SMEM, st>>>(p);
      else if (world <= 4) rs_adam_bulk_kernel<4, MODE><<<ctas, RSB_THREADS, RsBulk<4, ACC>::SMEM, st>>>(p);
      else rs_adam_bulk_kernel<MAXW, MODE><<<ctas, RSB_THREADS, RsBulk<MAXW, ACC>::SMEM, st>>>(p);
      return;
    }
    if (world == 1) rs_adam_kernel<1, MODE><<<ctas, threads, 0, st>>>(p);
    else if (world == 2) rs_adam_kernel<2, MODE><<<ctas, threads, 0, st>>>(p);
    else if (world <= 4) rs_adam_kernel<4, MODE><<<ctas, threads, 0, st>>>(p);
    else rs_adam_kernel<MAXW, MODE><<<ctas, threads, 0, st>>>(p);
  };
  switch (mode) {
    case RS_UPDATE: launch(std::integral_constant<int, RS_UPDATE>{}); break;
    case RS_FIRST: launch(std::integral_constant<int, RS_FIRST>{}); break;
    case RS_ADD: launch(std::integral_constant<int, RS_ADD>{}); break;
    default: launch(std::integral_constant<int, RS_FINAL>{}); break;
  }
  if (cudaGetLastError() != cudaSuccess) return DC_ECUDA;
  count_launch();
  return DC_OK;
}

struct PeerFlagsArg { uint32_t* p[MAXW]; int n; };
__global__ void set_scalars_kernel(float* dst, float s, float c) {
  dst[0] = s;
  dst[1] = c;
}
void k_set_scalars(float* dst, float s, float c, cudaStream_t st) {
  set_scalars_kernel<<<1, 1, 0, st>>>(dst, s, c);
  count_launch();
}

__global__ void inc_dev_kernel(uint32_t* dep) { *dep += 1u; }
__global__ void post_dev_kernel(const PeerFlagsArg d, const uint32_t* dep) {
  const uint32_t v = *reinterpret_cast<const volatile uint32_t*>(dep);
  __threadfence_system();
  for (int i = 0; i < d.n; ++i) ptx::st_release_sys(d.p[i], v);
}
__global__ void wait_dev_kernel(const uint32_t* f, int n, const uint32_t* dep, uint64_t tmo, uint32_t* err) {
  const uint32_t target = *reinterpret_cast<const volatile uint32_t*>(dep);
  const uint64_t t0 = ptx::globaltimer();
  for (int i = 0; i < n; ++i)
    if (!spin_ge(f + i, target, t0, tmo, err, 0x500u | i)) return;
}
void k_inc_dev(uint32_t* dep, cudaStream_t st) {
  inc_dev_kernel<<<1, 1, 0, st>>>(dep);
  count_launch();
}
void k_post_dev(PeerFlags dst, const uint32_t* dep, cudaStream_t st) {
  PeerFlagsArg a{};
  a.n = dst.n;
  for (int i = 0; i < dst.n; ++i) a.p[i] = dst.p[i];
  post_dev_kernel<<<1, 1, 0, st>>>(a, dep);
  count_launch();
}
void k_wait_dev(const uint32_t* flags, int n, const uint32_t* dep, uint64_t timeout_ns, uint32_t* err_flag,
                cudaStream_t st) {
  wait_dev_kernel<<<1, 1, 0, st>>>(flags, n, dep, timeout_ns, err_flag);
  count_launch();
}
void record_event(cudaEvent_t ev, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
  else cudaEventRecord(ev, st);
}

// ------------------------------------------------------------------ flags
struct PostParams { uint32_t* p[MAXW]; int n; uint32_t value; };
// +value on every listed counter (release, system scope) after the stream's
// earlier copies completed: the copy-engine gather's "my stores landed"
__global__ void add_flags_kernel(const PostParams p) {
  __threadfence_system();
  for (int i = 0; i < p.n; ++i) ptx::red_add_release_sys(p.p[i], p.value);
}

// Copy-engine all-gather: the same protocol as ag_push (wait
// every receiver's ready flag, then every sender bumps every receiver's done
// counter by one, then wait for N bumps per epoch) with the stores issued as
// cudaMemcpyAsync peer copies on the stream — no SM time for the data.
dc_status k_ag_copy(const std::vector<AgMember>& mem, int world, const uint64_t* arena_peers,
                    const uint32_t* ready_local, uint32_t epoch, PeerFlags done_peers, const uint32_t* done_local,
                    uint32_t done_target, uint64_t timeout_ns, uint32_t* err_flag, cudaStream_t st,
                    cudaEvent_t ev_after_ready) {
  wait_flags_kernel<<<1, 1, 0, st>>>(ready_local, world, epoch, timeout_ns, err_flag, 0x100u);
  count_launch();
  if (ev_after_ready) record_event(ev_after_ready, st);
  for (const AgMember& a : mem)
    for (int q = 0; q < world; ++q)
      if (cudaMemcpyAsync(reinterpret_cast<uint8_t*>(arena_peers[q]) + a.dst_off_bytes, a.src, a.bytes,
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return DC_ECUDA;
  PostParams p{};
  p.n = world;
  for (int q = 0; q < world; ++q) p.p[q] = done_peers.p[q];
  p.value = 1;
  add_flags_kernel<<<1, 1, 0, st>>>(p);
  count_launch();
  wait_flags_kernel<<<1, 1, 0, st>>>(done_local, 1, done_target, timeout_ns, err_flag, 0x200u);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? DC_OK : DC_ECUDA;
}

__global__ void post_flags_kernel(const PostParams p) {
  __threadfence_system();
  for (int i = 0; i < p.n; ++i) ptx::st_release_sys(p.p[i], p.value);
}
void k_delay(uint32_t us, cudaStream_t st) {
  if (!us) return;
  delay_kernel<<<1, 1, 0, st>>>(us);
  count_launch();
}

void k_post_flags(PeerFlags dst, uint32_t value, cudaStream_t st) {
  PostParams p{};
  p.n = dst.n;
  for (int i = 0; i < dst.n; ++i) p.p[i] = dst.p[i];
  p.value = value;
  post_flags_kernel<<<1, 1, 0, st>>>(p);
  count_launch();
}

void k_wait_flags(const uint32_t* flags, int n, uint32_t target, uint64_t timeout_ns, uint32_t* err_flag,
                  cudaStream_t st) {
  wait_flags_kernel<<<1, 1, 0, st>>>(flags, n, target, timeout_ns, err_flag, 0x400u);
  count_launch();
}

}  // namespace dc

namespace dc {
// Force-load this file's kernels (CUDA lazy loading would otherwise load a
// kernel at its first launch, which can block behind a spinning flag wait of
// another rank sharing the GPU).
cudaError_t preload_comm_kernels() {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, ag_push_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, ag_push_chunked_kernel);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(ag_push_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, AGB_SMEM);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, delay_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, wait_flags_kernel);
  auto pre_bulk = [&](auto mode_c) {
    constexpr int MODE = decltype(mode_c)::value;
    constexpr bool ACC = MODE == RS_FINAL;
#define DC_RSB_ATTR(Q)                                                                              \
    if (e == cudaSuccess)                                                                           \
      e = cudaFuncSetAttribute(rs_adam_bulk_kernel<Q, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               RsBulk<Q, ACC>::SMEM);
    DC_RSB_ATTR(1) DC_RSB_ATTR(2) DC_RSB_ATTR(4) DC_RSB_ATTR(MAXW)
#undef DC_RSB_ATTR
  };
  pre_bulk(std::integral_constant<int, RS_UPDATE>{});
  pre_bulk(std::integral_constant<int, RS_FINAL>{});
  auto pre = [&](auto mode_c) {
    constexpr int MODE = decltype(mode_c)::value;
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, rs_adam_kernel<1, MODE>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, rs_adam_kernel<2, MODE>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, rs_adam_kernel<4, MODE>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, rs_adam_kernel<MAXW, MODE>);
  };
  pre(std::integral_constant<int, RS_UPDATE>{});
  pre(std::integral_constant<int, RS_FIRST>{});
  pre(std::integral_constant<int, RS_ADD>{});
  pre(std::integral_constant<int, RS_FINAL>{});
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, post_flags_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, add_flags_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, set_scalars_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, inc_dev_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, post_dev_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, wait_dev_kernel);
  return e;
}
}  // namespace dc
