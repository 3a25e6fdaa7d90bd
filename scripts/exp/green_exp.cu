// Experiment: SM partitioning with green contexts.  GEMM (libdc_b200 dc_gemm,
// pair kernel) on a 128-SM partition while an Adam-like streaming kernel runs
// on a small partition.  Prints times / bandwidths.  Not part of the library.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../include/dc.h"

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); printf("CU error %s at %d\n", s, __LINE__); exit(1);} } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(r_), __LINE__); exit(1);} } while (0)

__global__ void fill_random(uint16_t* x, int64_t n, uint32_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed; h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    // bf16 in [-1, 1): sign, exponent 119..126, random mantissa
    x[i] = (uint16_t)(((h & 1) << 15) | ((119 + (h >> 1) % 8) << 7) | ((h >> 8) & 0x7f));
  }
}

__global__ void smid_kernel(int* out) {
  if (threadIdx.x == 0) { int s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); atomicOr(out + s, 1); }
}

// read g (bf16) + p, m, v (fp32); write p, m, v — 26 B per element
__global__ void __launch_bounds__(256) stream_kernel(const __nv_bfloat16* __restrict__ g, float* p, float* m, float* v, int64_t n) {
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n / 4; i += nthr) {
    float4 pp = reinterpret_cast<float4*>(p)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    uint2 gg = reinterpret_cast<const uint2*>(g)[i];
    float gf = __bfloat162float(*reinterpret_cast<__nv_bfloat16*>(&gg.x));
    mm.x = mm.x * 0.9f + gf; mm.y *= 0.9f; mm.z *= 0.9f; mm.w *= 0.9f;
    vv.x = vv.x * 0.999f + gf * gf; vv.y *= 0.999f; vv.z *= 0.999f; vv.w *= 0.999f;
    pp.x -= 1e-3f * mm.x; pp.y -= 1e-3f * mm.y; pp.z -= 1e-3f * mm.z; pp.w -= 1e-3f * mm.w;
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
  }
}

int main(int argc, char** argv) {
  const int n_small = argc > 1 ? atoi(argv[1]) : 16;
  const int gemm_sms_arg = argc > 2 ? atoi(argv[2]) : 0;
  const int Marg = argc > 3 ? atoi(argv[3]) : 4096, Narg = argc > 4 ? atoi(argv[4]) : 14336, Karg = argc > 5 ? atoi(argv[5]) : 4096;
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs %u\n", all.sm.smCount);
  // split: one group of n_small SMs, the remainder for the GEMM
  CUdevResource small_g, rest; unsigned nb = 1;
  CK(cuDevSmResourceSplitByCount(&small_g, &nb, &all, &rest, 0, n_small));
  printf("small %u rest %u\n", small_g.sm.smCount, rest.sm.smCount);
  CUdevResourceDesc d_small, d_rest;
  CK(cuDevResourceGenerateDesc(&d_small, &small_g, 1));
  CK(cuDevResourceGenerateDesc(&d_rest, &rest, 1));
  CUgreenCtx g_small, g_rest;
  CK(cuGreenCtxCreate(&g_small, d_small, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&g_rest, d_rest, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream s_small, s_rest;
  CK(cuGreenCtxStreamCreate(&s_small, g_small, CU_STREAM_NON_BLOCKING, 0));
  CK(cuGreenCtxStreamCreate(&s_rest, g_rest, CU_STREAM_NON_BLOCKING, 0));
  // memory from the primary context (runtime)
  int* smids; RK(cudaMalloc(&smids, 2 * 256 * 4)); RK(cudaMemset(smids, 0, 2 * 256 * 4));
  smid_kernel<<<1000, 32, 0, (cudaStream_t)s_small>>>(smids);
  smid_kernel<<<1000, 32, 0, (cudaStream_t)s_rest>>>(smids + 256);
  RK(cudaDeviceSynchronize());
  std::vector<int> h(512); RK(cudaMemcpy(h.data(), smids, 2048, cudaMemcpyDeviceToHost));
  int c0 = 0, c1 = 0, both = 0;
  for (int i = 0; i < 256; ++i) { c0 += h[i]; c1 += h[256 + i]; both += h[i] & h[256 + i]; }
  printf("SMs used: small-ctx %d, rest-ctx %d, overlap %d\n", c0, c1, both);

  // GEMM operands (down dX shape: M 4096, N 14336, K 4096, fwd layout)
  const int M = Marg, N = Narg, K = Karg;
  __nv_bfloat16 *A, *B, *C;
  RK(cudaMalloc(&A, (size_t)M * K * 2)); RK(cudaMalloc(&B, (size_t)N * K * 2)); RK(cudaMalloc(&C, (size_t)M * N * 2));
  fill_random<<<1184, 256>>>((uint16_t*)A, (int64_t)M * K, 1); fill_random<<<1184, 256>>>((uint16_t*)B, (int64_t)N * K, 2);
  dc_gemm_args ga{};
  ga.M = M; ga.N = N; ga.K = K; ga.A = A; ga.lda = K; ga.n_bseg = 1; ga.B[0] = B; ga.ldb[0] = K;
  ga.bseg_end[0] = N / 256; ga.C = C; ga.ldc = N; ga.kernel = 2;
  // streaming arrays: 218 M elements (one Llama-8B layer's shard at N = 1)
  const int64_t ne = 218ll * 1000 * 1000;
  __nv_bfloat16* g; float *p, *m, *v;
  RK(cudaMalloc(&g, ne * 2)); RK(cudaMalloc(&p, ne * 4)); RK(cudaMalloc(&m, ne * 4)); RK(cudaMalloc(&v, ne * 4));
  fill_random<<<1184, 256>>>((uint16_t*)g, ne, 3); fill_random<<<1184, 256>>>((uint16_t*)p, 2 * ne, 4);
  fill_random<<<1184, 256>>>((uint16_t*)m, 2 * ne, 5); fill_random<<<1184, 256>>>((uint16_t*)v, 2 * ne, 6);
  cudaEvent_t e0, e1, f0, f1;
  RK(cudaEventCreate(&e0)); RK(cudaEventCreate(&e1)); RK(cudaEventCreate(&f0)); RK(cudaEventCreate(&f1));
  auto run_gemm = [&](cudaStream_t st, int sms, int reps) {
    ga.num_sms = sms;
    for (int i = 0; i < reps; ++i) if (dc_gemm(&ga, st) != DC_OK) { printf("gemm failed\n"); exit(1); }
  };
  auto run_stream = [&](cudaStream_t st, int ctas, int reps) {
    for (int i = 0; i < reps; ++i) stream_kernel<<<ctas, 256, 0, st>>>(g, p, m, v, ne);
  };
  const double gflop = 2.0 * M * N * K / 1e9, gbytes = 26.0 * ne / 1e9;
  float ms;
  RK(cudaDeviceSynchronize());
  for (int pass = 0; pass < 2; ++pass) {
    // (d) full GPU, primary stream
    run_gemm(0, 0, 3); RK(cudaDeviceSynchronize());
    RK(cudaEventRecord(e0, 0)); run_gemm(0, 0, 40); RK(cudaEventRecord(e1, 0)); RK(cudaEventSynchronize(e1));
    RK(cudaEventElapsedTime(&ms, e0, e1)); printf("GEMM full GPU (148): %.1f TFLOP/s\n", gflop * 40 / ms);
    // (a) rest partition alone
    const int rest_sms = gemm_sms_arg ? gemm_sms_arg : (int)rest.sm.smCount;
    cudaStream_t sr = (cudaStream_t)s_rest, ss = (cudaStream_t)s_small;
    run_gemm(sr, rest_sms, 3); RK(cudaDeviceSynchronize());
    RK(cudaEventRecord(e0, sr)); run_gemm(sr, rest_sms, 40); RK(cudaEventRecord(e1, sr)); RK(cudaEventSynchronize(e1));
    RK(cudaEventElapsedTime(&ms, e0, e1)); printf("GEMM rest ctx (%d): %.1f TFLOP/s\n", rest_sms, gflop * 40 / ms);
    // (b) stream alone on small partition
    for (int ctas : {n_small * 2, n_small * 4, n_small * 8}) {
      run_stream(ss, ctas, 1); RK(cudaDeviceSynchronize());
      RK(cudaEventRecord(f0, ss)); run_stream(ss, ctas, 5); RK(cudaEventRecord(f1, ss)); RK(cudaEventSynchronize(f1));
      RK(cudaEventElapsedTime(&ms, f0, f1)); printf("stream small ctx, %d CTAs: %.1f GB/s\n", ctas, gbytes * 5 / ms * 1e3);
    }
    // (b') stream alone on full GPU
    run_stream(0, 296, 1); RK(cudaDeviceSynchronize());
    RK(cudaEventRecord(f0, 0)); run_stream(0, 296, 5); RK(cudaEventRecord(f1, 0)); RK(cudaEventSynchronize(f1));
    RK(cudaEventElapsedTime(&ms, f0, f1)); printf("stream full GPU: %.1f GB/s\n", gbytes * 5 / ms * 1e3);
    // (c) concurrent
    RK(cudaDeviceSynchronize());
    RK(cudaEventRecord(e0, sr)); run_gemm(sr, rest_sms, 40); RK(cudaEventRecord(e1, sr));
    RK(cudaEventRecord(f0, ss)); run_stream(ss, n_small * 8, 8); RK(cudaEventRecord(f1, ss));
    RK(cudaDeviceSynchronize());
    float ms2;
    RK(cudaEventElapsedTime(&ms, e0, e1)); RK(cudaEventElapsedTime(&ms2, f0, f1));
    printf("CONCURRENT: GEMM %.1f TFLOP/s (%.2f ms), stream %.1f GB/s (%.2f ms)\n", gflop * 40 / ms, ms,
           gbytes * 8 / ms2 * 1e3, ms2);
  }
  return 0;
}
