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
    for (int i = 0; i < count; ++i) add_stream_pair(nullptr, 0);
    return;
  }
  int total = 0;
  GMI_CUDA_CHECK(cudaDeviceGetAttribute(&total, cudaDevAttrMultiProcessorCount, device));
  const int per = sm_per_gmi > 0 ? sm_per_gmi : (total / count) / 8 * 8;
  make_green(device, std::vector<int>(count, per));
}

GmiResources::GmiResources(int device, const std::vector<int>& sms, int backend) : backend_(backend) {
  GMI_CUDA_CHECK(cudaSetDevice(device));
  if (backend == 0) {
    for (size_t i = 0; i < sms.size(); ++i) add_stream_pair(nullptr, 0);
    return;
  }
  make_green(device, sms);
}

void GmiResources::add_stream_pair(void* green, int sms) {
  if (!green) {
    cudaStream_t s;
    GMI_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    streams_.push_back(s);
    GMI_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    aux_.push_back(s);
    sms_.push_back(sms);
    return;
  }
  using StreamCreate = CUresult (*)(CUstream*, CUgreenCtx, unsigned, int);
  static auto cuGreenCtxStreamCreate_ = driver_fn<StreamCreate>("cuGreenCtxStreamCreate");
  CUstream s;
  cu_check(cuGreenCtxStreamCreate_(&s, static_cast<CUgreenCtx>(green), CU_STREAM_NON_BLOCKING, 0),
           "cuGreenCtxStreamCreate");
  streams_.push_back(reinterpret_cast<cudaStream_t>(s));
  cu_check(cuGreenCtxStreamCreate_(&s, static_cast<CUgreenCtx>(green), CU_STREAM_NON_BLOCKING, 0),
           "cuGreenCtxStreamCreate");
  aux_.push_back(reinterpret_cast<cudaStream_t>(s));
  sms_.push_back(sms);
}

// One SM group per GMI, carved off the device's SM resource in order
// (cuDevSmResourceSplitByCount with a single group of the requested size, then the remainder
// is split again); an entry of 0 takes whatever the other GMIs left over.
void GmiResources::make_green(int device, const std::vector<int>& sms) {
  using GetDev = CUresult (*)(CUdevice*, int);
  using GetRes = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
  using Split = CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned);
  using GenDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned);
  using Create = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
  auto cuDeviceGet_ = driver_fn<GetDev>("cuDeviceGet");
  auto cuDeviceGetDevResource_ = driver_fn<GetRes>("cuDeviceGetDevResource");
  auto cuDevSmResourceSplitByCount_ = driver_fn<Split>("cuDevSmResourceSplitByCount");
  auto cuDevResourceGenerateDesc_ = driver_fn<GenDesc>("cuDevResourceGenerateDesc");
  auto cuGreenCtxCreate_ = driver_fn<Create>("cuGreenCtxCreate");

  GMI_CUDA_CHECK(cudaFree(nullptr));  // make the primary context current first
  CUdevice dev;
  cu_check(cuDeviceGet_(&dev, device), "cuDeviceGet");
  CUdevResource all{};
  cu_check(cuDeviceGetDevResource_(dev, &all, CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource");
  const int total = int(all.sm.smCount);
  int fixed = 0, zeros = 0;
  for (int s : sms) {
    if (s == 0) ++zeros;
    else if (s < 8 || s % 8 != 0) fail(GMI_ERR_INVALID, "green-context GMI sizes must be multiples of 8 SMs (>= 8)");
    fixed += s;
  }
  if (zeros > 1 || fixed > total || (zeros == 1 && total - fixed < 8))
    fail(GMI_ERR_INVALID, "green-context split infeasible: " + std::to_string(sms.size()) + " GMIs, " +
                              std::to_string(fixed) + " fixed SMs on a " + std::to_string(total) + "-SM GPU");
  std::vector<CUdevResource> res(sms.size());
  bool equal = zeros == 0;
  for (int s : sms) equal = equal && s == sms[0];
  if (equal) {  // one split call: the driver places the equal groups itself
    unsigned n = unsigned(sms.size());
    CUdevResource rest{};
    cu_check(cuDevSmResourceSplitByCount_(res.data(), &n, &all, &rest, 0, unsigned(sms[0])),
             "cuDevSmResourceSplitByCount");
    if (n < sms.size()) fail(GMI_ERR_INVALID, "green-context split produced too few groups");
  } else {
    CUdevResource cur = all;
    for (size_t i = 0; i < sms.size(); ++i) {
      if (sms[i] == 0) continue;
      unsigned n = 1;
      CUdevResource rest{};
      cu_check(cuDevSmResourceSplitByCount_(&res[i], &n, &cur, &rest, 0, unsigned(sms[i])),
               "cuDevSmResourceSplitByCount");
      if (n < 1) fail(GMI_ERR_INVALID, "green-context split produced no group");
      cur = rest;
    }
    for (size_t i = 0; i < sms.size(); ++i)
      if (sms[i] == 0) res[i] = cur;
  }
  for (size_t i = 0; i < sms.size(); ++i) {
    CUdevResourceDesc desc;
    cu_check(cuDevResourceGenerateDesc_(&desc, &res[i], 1), "cuDevResourceGenerateDesc");
    CUgreenCtx g;
    cu_check(cuGreenCtxCreate_(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
    green_.push_back(g);
    add_stream_pair(g, int(res[i].sm.smCount));
  }
}

cudaStream_t GmiResources::extra_stream(int i) {
  const size_t n = streams_.size();
  add_stream_pair(green_.empty() ? nullptr : green_.at(i), sms_.at(i));
  cudaStream_t s = streams_.back();
  // keep the per-GMI vectors indexed by GMI: the new pair lives past the GMIs
  extra_.push_back(streams_.back());
  extra_.push_back(aux_.back());
  streams_.resize(n);
  aux_.resize(n);
  sms_.resize(n);
  return s;
}

GmiResources::~GmiResources() {
  for (auto s : extra_) cudaStreamDestroy(s);
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
