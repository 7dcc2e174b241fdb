// K1: intra-GPU GMI gradient reduction over shared device buffers.
//
// GMIs are green-context partitions of one process, so their gradient buffers live in
// one address space: the reference's host-bounce rings (reduction.hpp:170-212) collapse
// into one HBM-bound pass. To stay bit-identical to the reference's result, every element
// is folded in exactly the order its ring schedule would have accumulated it: element e
// belongs to chunk c = the c with len*c/n <= e < len*(c+1)/n (reduction.hpp:164-166), and
// that chunk's running sum starts at ring member c and picks up members c+1, c+2, ... in
// ring order. MRR sums the per-ring results into a zero-initialised total in ring order
// (reduction.hpp:271-275); HAR folds per-GPU rings first, then the leaders' ring over GPUs.
//
// Traffic per call: n reads + 1 write (+ n writes when broadcasting) of len elements.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "../host/errors.hpp"
#include "../host/planner.hpp"
#include "launch.cuh"

namespace gmi {

using u64 = unsigned long long;

constexpr int kMaxReduceBufs = 128;
constexpr int kMaxReduceGpus = 32;

struct ReduceArgs {
  const void* bufs[kMaxReduceBufs];  // flattened layout order
  void* out;
  int algo, g, n, t, broadcast;
  u64 len;
  int counts[kMaxReduceGpus];
  int offs[kMaxReduceGpus];
  unsigned char ring[kMaxReduceBufs];  // MRR: ring r member j -> flat index, at r*g + j
};

__device__ __forceinline__ int chunk_of(u64 e, u64 len, int n) {
  return int(((e + 1) * u64(n) + len - 1) / len) - 1;
}

// Fold of `e` over members idx[0..n) in ring order starting at chunk owner c.
template <typename T>
__device__ __forceinline__ T ring_fold(const ReduceArgs& a, const unsigned char* idx, const int* span_idx,
                                       int n, u64 e) {
  const int c = chunk_of(e, a.len, n);
  auto at = [&](int k) -> int { return idx ? int(idx[k]) : span_idx[0] + k; };
  T acc = static_cast<const T*>(a.bufs[at(c)])[e];
  for (int j = 1; j < n; ++j) {
    int k = c + j;
    if (k >= n) k -= n;
    acc = static_cast<const T*>(a.bufs[at(k)])[e] + acc;
  }
  return acc;
}

template <typename T>
__global__ void __launch_bounds__(256) gmi_reduce_kernel(const __grid_constant__ ReduceArgs a) {
  pdl_trigger();
  pdl_wait();
  const u64 stride = u64(gridDim.x) * blockDim.x;
  for (u64 e = u64(blockIdx.x) * blockDim.x + threadIdx.x; e < a.len; e += stride) {
    T acc;
    if (a.algo == 0) {  // MPR: one ring over every GMI, flattened order
      const int zero = 0;
      acc = ring_fold<T>(a, nullptr, &zero, a.n, e);
    } else if (a.algo == 1) {  // MRR: t disjoint rings of g, then endpoint total
      if (a.g < 2) {
        acc = static_cast<const T*>(a.bufs[a.ring[0]])[e];
      } else {
        acc = T(0);
        for (int r = 0; r < a.t; ++r) acc = acc + ring_fold<T>(a, a.ring + r * a.g, nullptr, a.g, e);
      }
    } else {  // HAR: per-GPU rings, then the leaders' ring in GPU order
      const int c = chunk_of(e, a.len, a.g);
      acc = ring_fold<T>(a, nullptr, &a.offs[c], a.counts[c], e);
      for (int j = 1; j < a.g; ++j) {
        int k = c + j;
        if (k >= a.g) k -= a.g;
        acc = ring_fold<T>(a, nullptr, &a.offs[k], a.counts[k], e) + acc;
      }
    }
    static_cast<T*>(a.out)[e] = acc;
    if (a.broadcast)
      for (int i = 0; i < a.n; ++i) const_cast<T*>(static_cast<const T*>(a.bufs[i]))[e] = acc;
  }
}

void reduce_device(plan::Algo algo, const plan::Placement& p, void* const* bufs, void* out, size_t len,
                   int dtype, bool broadcast, cudaStream_t stream) {
  p.check();
  ReduceArgs a{};
  const auto flat = p.flat();
  if (int(flat.size()) > kMaxReduceBufs) invalid("too many GMIs for one device reduction");
  if (p.gpus() > kMaxReduceGpus) invalid("too many GPUs for one device reduction");
  if (!out) invalid("null output buffer");
  a.n = int(flat.size());
  a.g = p.gpus();
  a.algo = int(algo);
  a.len = len;
  a.out = out;
  a.broadcast = broadcast ? 1 : 0;
  for (int i = 0; i < a.n; ++i) {
    if (!bufs[i]) invalid("null GMI buffer");
    a.bufs[i] = bufs[i];
  }
  int off = 0;
  for (int gpu = 0; gpu < a.g; ++gpu) {
    a.counts[gpu] = int(p.per_gpu[gpu].size());
    a.offs[gpu] = off;
    off += a.counts[gpu];
  }
  if (algo == plan::Algo::MRR) {
    const auto rings = plan::disjoint_rings(p);  // throws MULTISTREAM like the reference
    a.t = int(rings.size());
    for (int r = 0; r < a.t; ++r)
      for (int j = 0; j < a.g; ++j) {
        const int id = rings[r][j];
        a.ring[r * a.g + j] = static_cast<unsigned char>(std::find(flat.begin(), flat.end(), id) - flat.begin());
      }
  }
  if (len == 0) return;
  const int threads = 256;
  const u64 want = (len + threads - 1) / threads;
  const int blocks = int(std::min<u64>(want, 148ull * 16));
  if (dtype == GMI_F64)
    launch_pdl(gmi_reduce_kernel<double>, dim3(blocks), dim3(threads), 0, stream, a);
  else if (dtype == GMI_F32)
    launch_pdl(gmi_reduce_kernel<float>, dim3(blocks), dim3(threads), 0, stream, a);
  else
    invalid("dtype must be GMI_F32 or GMI_F64");
}

}  // namespace gmi

extern "C" GMI_API int gmi_execute_host(int strategy, int num_gpus, const int* counts, const int* ids,
                                        const void* const* bufs, size_t len, int dtype, void* result) {
  return gmi::guarded([&] {
    if (strategy < 0 || strategy > 2) gmi::invalid("unknown strategy");
    if (dtype != GMI_F32 && dtype != GMI_F64) gmi::invalid("dtype must be GMI_F32 or GMI_F64");
    gmi::plan::Placement p;
    if (num_gpus < 0) gmi::invalid("num_gpus must be >= 0");
    p.per_gpu.resize(num_gpus);
    int k = 0;
    for (int g = 0; g < num_gpus; ++g) {
      p.per_gpu[g].assign(ids + k, ids + k + counts[g]);
      k += counts[g];
    }
    p.check();
    const size_t esz = dtype == GMI_F64 ? 8 : 4;
    const size_t n = p.flat().size();
    const size_t bytes = std::max<size_t>(len * esz, 16);
    char* arena = nullptr;
    GMI_CUDA_CHECK(cudaMalloc(&arena, bytes * (n + 1)));
    std::vector<void*> dev(n);
    cudaStream_t s = nullptr;
    try {
      GMI_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      for (size_t i = 0; i < n; ++i) {
        dev[i] = arena + i * bytes;
        GMI_CUDA_CHECK(cudaMemcpyAsync(dev[i], bufs[i], len * esz, cudaMemcpyHostToDevice, s));
      }
      gmi::reduce_device(gmi::plan::Algo(strategy), p, dev.data(), arena + n * bytes, len, dtype, false, s);
      GMI_CUDA_CHECK(cudaMemcpyAsync(result, arena + n * bytes, len * esz, cudaMemcpyDeviceToHost, s));
      GMI_CUDA_CHECK(cudaStreamSynchronize(s));
    } catch (...) {
      if (s) cudaStreamDestroy(s);
      cudaFree(arena);
      throw;
    }
    cudaStreamDestroy(s);
    cudaFree(arena);
  });
}

extern "C" GMI_API int gmi_reduce_device(int strategy, int num_gpus, const int* counts, const int* ids,
                                         void* const* bufs, void* out, size_t len, int dtype, int broadcast,
                                         void* stream) {
  return gmi::guarded([&] {
    if (strategy < 0 || strategy > 2) gmi::invalid("unknown strategy");
    gmi::plan::Placement p;
    if (num_gpus < 0) gmi::invalid("num_gpus must be >= 0");
    p.per_gpu.resize(num_gpus);
    int k = 0;
    for (int g = 0; g < num_gpus; ++g) {
      p.per_gpu[g].assign(ids + k, ids + k + counts[g]);
      k += counts[g];
    }
    gmi::reduce_device(gmi::plan::Algo(strategy), p, bufs, out, len, dtype, broadcast != 0,
                       static_cast<cudaStream_t>(stream));
  });
}

extern "C" GMI_API int gmi_allreduce(int strategy, int num_gpus, const int* counts, const int* ids,
                                     void* const* dev_bufs, size_t len, int dtype, void* const* streams, double b1,
                                     double b2, gmi_reduction_info_t* run) {
  return gmi::guarded([&] {
    if (strategy < 0 || strategy > 2) gmi::invalid("unknown strategy");
    if (dtype != GMI_F32 && dtype != GMI_F64) gmi::invalid("dtype must be GMI_F32 or GMI_F64");
    if (!dev_bufs) gmi::invalid("null buffer list");
    gmi::plan::Placement p;
    if (num_gpus < 0) gmi::invalid("num_gpus must be >= 0");
    p.per_gpu.resize(num_gpus);
    int k = 0;
    for (int g = 0; g < num_gpus; ++g) {
      p.per_gpu[g].assign(ids + k, ids + k + counts[g]);
      k += counts[g];
    }
    p.check();
    const size_t n = p.flat().size();
    if (run) {  // the reference's accounting of the same call (fp64 bytes, as execute() counts them)
      const int rc = gmi_reduction_schedule(strategy, num_gpus, counts, ids, len, 8.0, b1, b2, nullptr, 0, run);
      if (rc != 0) gmi::fail(rc, gmi_last_error());
    }
    cudaStream_t s0 = streams ? static_cast<cudaStream_t>(streams[0]) : nullptr;
    // every GMI stream reaches the call before the fold reads its buffer ...
    std::vector<cudaEvent_t> evs;
    auto event = [&] {
      cudaEvent_t e = nullptr;
      GMI_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      evs.push_back(e);
      return e;
    };
    try {
      for (size_t i = 1; streams && i < n; ++i) {
        cudaStream_t si = static_cast<cudaStream_t>(streams[i]);
        if (si == s0) continue;
        cudaEvent_t e = event();
        GMI_CUDA_CHECK(cudaEventRecord(e, si));
        GMI_CUDA_CHECK(cudaStreamWaitEvent(s0, e, 0));
      }
      // ... the fold writes the total into every buffer (the first one is also the output: the
      // kernel is elementwise, each element read from every buffer before it is written) ...
      gmi::reduce_device(gmi::plan::Algo(strategy), p, dev_bufs, dev_bufs[0], len, dtype, true, s0);
      // ... and every GMI stream continues after it
      if (streams && n > 1) {
        cudaEvent_t done = event();
        GMI_CUDA_CHECK(cudaEventRecord(done, s0));
        for (size_t i = 1; i < n; ++i)
          if (static_cast<cudaStream_t>(streams[i]) != s0)
            GMI_CUDA_CHECK(cudaStreamWaitEvent(static_cast<cudaStream_t>(streams[i]), done, 0));
      }
    } catch (...) {
      for (cudaEvent_t e : evs) cudaEventDestroy(e);
      throw;
    }
    for (cudaEvent_t e : evs) cudaEventDestroy(e);  // released once the recorded work completes
  });
}
