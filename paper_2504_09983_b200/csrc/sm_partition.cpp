// Spatial SM partition for one rank's step (CUDA green contexts): a GEMM
// partition and a small communication / optimizer partition, each with its
// own streams.  The HBM-bound reduce-scatter + Adam (and the NVLink gathers at
// N > 1) then run truly beside the tensor-bound GEMMs instead of taking SMs
// from them wave by wave (profiles/r01e).  The driver entry
// points are resolved at run time (cudaGetDriverEntryPoint), so the library
// does not link libcuda.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>
#include <string>

#include "dc_internal.h"

namespace dc {

namespace {
using PFN_GetDevResource = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
using PFN_SplitByCount = CUresult (*)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*,
                                      unsigned int, unsigned int);
using PFN_GenerateDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned int);
using PFN_GreenCtxCreate = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
using PFN_GreenCtxDestroy = CUresult (*)(CUgreenCtx);
using PFN_GreenCtxStreamCreate = CUresult (*)(CUstream*, CUgreenCtx, unsigned int, int);

struct Driver {
  PFN_GetDevResource get_resource = nullptr;
  PFN_SplitByCount split = nullptr;
  PFN_GenerateDesc gen_desc = nullptr;
  PFN_GreenCtxCreate create = nullptr;
  PFN_GreenCtxDestroy destroy = nullptr;
  PFN_GreenCtxStreamCreate stream_create = nullptr;
  bool ok = false;
};

const Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn;
    };
    void* f[6] = {};
    d.ok = get("cuDeviceGetDevResource", &f[0]) && get("cuDevSmResourceSplitByCount", &f[1]) &&
           get("cuDevResourceGenerateDesc", &f[2]) && get("cuGreenCtxCreate", &f[3]) &&
           get("cuGreenCtxDestroy", &f[4]) && get("cuGreenCtxStreamCreate", &f[5]);
    d.get_resource = reinterpret_cast<PFN_GetDevResource>(f[0]);
    d.split = reinterpret_cast<PFN_SplitByCount>(f[1]);
    d.gen_desc = reinterpret_cast<PFN_GenerateDesc>(f[2]);
    d.create = reinterpret_cast<PFN_GreenCtxCreate>(f[3]);
    d.destroy = reinterpret_cast<PFN_GreenCtxDestroy>(f[4]);
    d.stream_create = reinterpret_cast<PFN_GreenCtxStreamCreate>(f[5]);
  });
  return d;
}
}  // namespace

dc_status sm_partition_create(int device, int comm_sms, SmPartition* out, std::string* err) {
  *out = SmPartition{};
  const Driver& d = driver();
  if (!d.ok) { *err = "green contexts unavailable in this driver"; return DC_ECUDA; }
  CUdevice dev = device;
  CUdevResource all{};
  if (d.get_resource(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) { *err = "cuDeviceGetDevResource failed"; return DC_ECUDA; }
  const int total = (int)all.sm.smCount;
  // GEMM partition: the largest multiple of 8 SMs (green-context granularity)
  // leaving at least comm_sms; the communication partition takes the rest
  const int gemm = (total - comm_sms) / 8 * 8;
  if (comm_sms < 1 || gemm < 16) { *err = "bad SM partition size"; return DC_EINVAL; }
  CUdevResource g{}, rest{};
  unsigned int nb = 1;
  if (d.split(&g, &nb, &all, &rest, 0, (unsigned)gemm) != CUDA_SUCCESS || nb != 1) {
    *err = "cuDevSmResourceSplitByCount failed";
    return DC_ECUDA;
  }
  CUdevResourceDesc dg = nullptr, dr = nullptr;
  CUgreenCtx cg = nullptr, cr = nullptr;
  if (d.gen_desc(&dg, &g, 1) != CUDA_SUCCESS || d.gen_desc(&dr, &rest, 1) != CUDA_SUCCESS ||
      d.create(&cg, dg, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      d.create(&cr, dr, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
    *err = "green context creation failed";
    return DC_ECUDA;
  }
  CUstream s0 = nullptr, s1 = nullptr, s2 = nullptr;
  if (d.stream_create(&s0, cg, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
      d.stream_create(&s1, cr, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
      d.stream_create(&s2, cr, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) {
    *err = "green context stream creation failed";
    return DC_ECUDA;
  }
  out->gemm_sms = (int)g.sm.smCount;
  out->comm_sms = (int)rest.sm.smCount;
  out->compute = reinterpret_cast<cudaStream_t>(s0);
  out->rs = reinterpret_cast<cudaStream_t>(s1);
  out->ag = reinterpret_cast<cudaStream_t>(s2);
  out->ctx_gemm = cg;
  out->ctx_comm = cr;
  return DC_OK;
}

void sm_partition_destroy(SmPartition* p) {
  if (!p || !p->ctx_gemm) return;
  const Driver& d = driver();
  cudaStreamDestroy(p->compute);
  cudaStreamDestroy(p->rs);
  cudaStreamDestroy(p->ag);
  d.destroy(reinterpret_cast<CUgreenCtx>(p->ctx_gemm));
  d.destroy(reinterpret_cast<CUgreenCtx>(p->ctx_comm));
  *p = SmPartition{};
}

}  // namespace dc
