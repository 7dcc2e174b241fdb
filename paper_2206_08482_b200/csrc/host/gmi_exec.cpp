// GMI execution resources. A GMI (GPU multiplexing instance) is realised either as a
// plain CUDA stream sharing all SMs, or as an SM-partitioned CUDA green context
// (cuDevSmResourceSplitByCount -> cuDevResourceGenerateDesc -> cuGreenCtxCreate ->
// cuGreenCtxStreamCreate) — the B200 counterpart of the reference's MPS share / MIG
// profile partitions (topology.hpp:72-88). All GMIs of a GPU live in one process, so
// device buffers are shared and inter-GMI traffic never bounces through the host.
#include "gmi_exec.hpp"

#include <cuda.h>

#include <string>

#include "errors.hpp"

namespace gmi {

namespace {

template <class Fn>
Fn driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    fail(GMI_ERR_CUDA, std::string("driver entry point unavailable: ") + name);
  return reinterpret_cast<Fn>(p);
}

void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) fail(GMI_ERR_CUDA, std::string(what) + " failed with CUresult " + std::to_string(int(r)));
}

}  // namespace

GmiResources::GmiResources(int device, int count, int backend, int sm_per_gmi) : backend_(backend) {
  GMI_CUDA_CHECK(cudaSetDevice(device));
  if (backend == 0) {
    for (int i = 0; i < count; ++i) {
      cudaStream_t s;
      GMI_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      streams_.push_back(s);
      GMI_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      aux_.push_back(s);
      sms_.push_back(0);
    }
    return;
  }
  using GetDev = CUresult (*)(CUdevice*, int);
  using GetRes = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
  using Split = CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned);
  using GenDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned);
  using Create = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
  using StreamCreate = CUresult (*)(CUstream*, CUgreenCtx, unsigned, int);
  auto cuDeviceGet_ = driver_fn<GetDev>("cuDeviceGet");
  auto cuDeviceGetDevResource_ = driver_fn<GetRes>("cuDeviceGetDevResource");
  auto cuDevSmResourceSplitByCount_ = driver_fn<Split>("cuDevSmResourceSplitByCount");
  auto cuDevResourceGenerateDesc_ = driver_fn<GenDesc>("cuDevResourceGenerateDesc");
  auto cuGreenCtxCreate_ = driver_fn<Create>("cuGreenCtxCreate");
  auto cuGreenCtxStreamCreate_ = driver_fn<StreamCreate>("cuGreenCtxStreamCreate");

  GMI_CUDA_CHECK(cudaFree(nullptr));  // make the primary context current first
  CUdevice dev;
  cu_check(cuDeviceGet_(&dev, device), "cuDeviceGet");
  CUdevResource all{};
  cu_check(cuDeviceGetDevResource_(dev, &all, CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource");
  const int total = int(all.sm.smCount);
  int per = sm_per_gmi > 0 ? sm_per_gmi : (total / count) / 8 * 8;
  if (per < 8 || per % 8 != 0 || per * count > total)
    fail(GMI_ERR_INVALID, "green-context split infeasible: " + std::to_string(count) + " GMIs x " +
                              std::to_string(per) + " SMs on a " + std::to_string(total) + "-SM GPU");
  std::vector<CUdevResource> groups(count);
  unsigned n = unsigned(count);
  CUdevResource rest{};
  cu_check(cuDevSmResourceSplitByCount_(groups.data(), &n, &all, &rest, 0, unsigned(per)),
           "cuDevSmResourceSplitByCount");
  if (int(n) < count) fail(GMI_ERR_INVALID, "green-context split produced too few groups");
  for (int i = 0; i < count; ++i) {
    CUdevResourceDesc desc;
    cu_check(cuDevResourceGenerateDesc_(&desc, &groups[i], 1), "cuDevResourceGenerateDesc");
    CUgreenCtx g;
    cu_check(cuGreenCtxCreate_(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
    CUstream s;
    cu_check(cuGreenCtxStreamCreate_(&s, g, CU_STREAM_NON_BLOCKING, 0), "cuGreenCtxStreamCreate");
    green_.push_back(g);
    streams_.push_back(reinterpret_cast<cudaStream_t>(s));
    cu_check(cuGreenCtxStreamCreate_(&s, g, CU_STREAM_NON_BLOCKING, 0), "cuGreenCtxStreamCreate");
    aux_.push_back(reinterpret_cast<cudaStream_t>(s));
    sms_.push_back(int(groups[i].sm.smCount));
  }
}

GmiResources::~GmiResources() {
  for (auto s : streams_) cudaStreamDestroy(s);
  for (auto s : aux_) cudaStreamDestroy(s);
  if (!green_.empty()) {
    using Destroy = CUresult (*)(CUgreenCtx);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuGreenCtxDestroy", &p, cudaEnableDefault, &q) == cudaSuccess && p)
      for (auto g : green_) reinterpret_cast<Destroy>(p)(static_cast<CUgreenCtx>(g));
  }
}

}  // namespace gmi
