// Ceiling of rs_adam's access pattern at N = 1 (experiment, not product code):
// per element read bf16 g + fp32 p, m, v and write fp32 p, m, v + bf16 shard
// (28 B), no Adam math.  (a) 16-byte LDG/STG grid-stride (rs_adam's pattern),
// (b) 1-D bulk async copies (cp.async.bulk) into shared memory, 3-stage ring,
// and bulk stores back.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 stream_mix.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>

__global__ void ldg_kernel(const uint4* __restrict__ g, uint4* p, uint4* m, uint4* v, uint2* sh, int64_t n8) {
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += 2 * nthr) {
    uint4 G[2], P[2][2], M[2][2], V[2][2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t j = i + u * nthr;
      if (j < n8) {
        G[u] = g[j];
        P[u][0] = p[2 * j]; P[u][1] = p[2 * j + 1];
        M[u][0] = m[2 * j]; M[u][1] = m[2 * j + 1];
        V[u][0] = v[2 * j]; V[u][1] = v[2 * j + 1];
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t j = i + u * nthr;
      if (j < n8) {
        P[u][0].x ^= G[u].x; M[u][0].y ^= G[u].y; V[u][1].z ^= G[u].z;
        p[2 * j] = P[u][0]; p[2 * j + 1] = P[u][1];
        m[2 * j] = M[u][0]; m[2 * j + 1] = M[u][1];
        v[2 * j] = V[u][0]; v[2 * j + 1] = V[u][1];
        sh[j] = make_uint2(P[u][0].x, P[u][0].y);
      }
    }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n .reg .pred P;\n W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W;\n}\n"
               :: "r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* s, const void* g, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(s)), "l"(g), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* s, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(g), "r"(smem_u32(s)), "r"(bytes)
               : "memory");
}

constexpr int CH = 2048;                 // elements per chunk
constexpr int ST = 3;                    // stages
constexpr int CHB = CH * 4 * 3 + CH * 2 + CH * 2;   // p m v fp32 + g bf16 + shard bf16

__global__ void __launch_bounds__(256) bulk_kernel(const char* g, char* p, char* m, char* v, char* sh, int64_t n) {
  extern __shared__ __align__(128) char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + ST * CHB);
  const int64_t nch = n / CH;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t c, int s) {
    char* b = smem + s * CHB;
    mbar_expect(&bar[s], CH * 14);
    bulk_g2s(b, p + c * CH * 4, CH * 4, &bar[s]);
    bulk_g2s(b + CH * 4, m + c * CH * 4, CH * 4, &bar[s]);
    bulk_g2s(b + CH * 8, v + c * CH * 4, CH * 4, &bar[s]);
    bulk_g2s(b + CH * 12, g + c * CH * 2, CH * 2, &bar[s]);
  };
  int64_t c0 = blockIdx.x;
  int k = 0;
  if (threadIdx.x == 0)
    for (int s = 0; s < ST - 1 && c0 + s * gridDim.x < nch; ++s) issue(c0 + s * gridDim.x, s);
  for (int64_t c = c0; c < nch; c += gridDim.x, ++k) {
    const int s = k % ST;
    const uint32_t ph = (k / ST) & 1;
    if (threadIdx.x == 0) {
      const int64_t cn = c + (int64_t)(ST - 1) * gridDim.x;
      if (cn < nch) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // stage (k-1)%ST stores drained
        issue(cn, (k + ST - 1) % ST);
      }
    }
    mbar_wait(&bar[s], ph);
    char* b = smem + s * CHB;
    uint32_t* P = reinterpret_cast<uint32_t*>(b);
    const uint32_t* G = reinterpret_cast<const uint32_t*>(b + CH * 12);
    uint32_t* S = reinterpret_cast<uint32_t*>(b + CH * 14);
    for (int i = threadIdx.x; i < CH / 2; i += blockDim.x) { P[2 * i] ^= G[i]; S[i] = P[2 * i]; }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_s2g(p + c * CH * 4, b, CH * 4);
      bulk_s2g(m + c * CH * 4, b + CH * 4, CH * 4);
      bulk_s2g(v + c * CH * 4, b + CH * 8, CH * 4);
      bulk_s2g(sh + c * CH * 2, b + CH * 14, CH * 2);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const int64_t n = 218LL << 20;          // ~ one Llama-3-8B layer (228 M elements)
  char *g, *p, *m, *v, *sh;
  cudaMalloc(&g, n * 2); cudaMalloc(&p, n * 4); cudaMalloc(&m, n * 4); cudaMalloc(&v, n * 4); cudaMalloc(&sh, n * 2);
  cudaMemset(g, 1, n * 2); cudaMemset(p, 0, n * 4); cudaMemset(m, 0, n * 4); cudaMemset(v, 0, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double bytes = 28.0 * n;
  for (int ctas : {296, 444}) {
    for (int r = 0; r < 2; ++r) ldg_kernel<<<ctas, 256>>>((const uint4*)g, (uint4*)p, (uint4*)m, (uint4*)v, (uint2*)sh, n / 8);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) ldg_kernel<<<ctas, 256>>>((const uint4*)g, (uint4*)p, (uint4*)m, (uint4*)v, (uint2*)sh, n / 8);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("ldg  ctas %d: %.3f ms  %.2f TB/s\n", ctas, ms / 5, bytes / (ms / 5 * 1e-3) / 1e12);
  }
  const int smem = ST * CHB + 64;
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int ctas : {148, 296}) {
    for (int r = 0; r < 2; ++r) bulk_kernel<<<ctas, 256, smem>>>(g, p, m, v, sh, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) bulk_kernel<<<ctas, 256, smem>>>(g, p, m, v, sh, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("bulk ctas %d (smem %d): %.3f ms  %.2f TB/s  err=%s\n", ctas, smem, ms / 5, bytes / (ms / 5 * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
