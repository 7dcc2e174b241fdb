// Measured profiler for the adaptive GMI manager (Alg. 2): the B200 implementation of the
// reference's Profiler::profile seam (search.hpp:32-37). Where the reference plugs in a
// SyntheticCostModel (search.hpp:100-132), this runs the real PPO iteration on this GPU with
// `gmis_per_gpu` GMIs (SM-partitioned green contexts or streams) of `num_env` environments
// each, using the catalog MLP of `bench` (workload.hpp:126-134), and reports per-GMI
// throughput (env-steps/s) and per-GMI device memory (GB). A configuration that cannot be
// built (partition too small, minibatch shape, out of memory) is reported as not runnable,
// which is how explore() prunes it.
#include <cuda_runtime.h>

#include <cstring>
#include <memory>

#include "errors.hpp"
#include "gmi.h"
#include "planner.hpp"
#include "trainer.hpp"

namespace gmi {

namespace {

struct ProbeSettings {
  int device, backend, iters;
};

void measure(const char* bench, int gpg, int num_env, const ProbeSettings& ps, int* runnable, double* top,
             double* mem) {
  *runnable = 0;
  *top = *mem = 0.0;
  if (!bench) invalid("null bench name");
  if (gpg < 1 || num_env < 1) invalid("profile needs gmis_per_gpu >= 1 and num_env >= 1");
  const plan::Workload w = plan::catalog(bench);  // rejects unknown names like the reference
  if (w.dims.size() < 3 || int(w.dims.size()) - 2 > GMI_MAX_HIDDEN) return;
  gmi_ppo_config_t c;
  gmi_ppo_config_defaults(&c);
  c.obs_dim = w.dims.front();
  c.act_dim = w.dims.back();
  c.num_hidden = int(w.dims.size()) - 2;
  for (int l = 0; l < c.num_hidden; ++l) c.hidden[l] = w.dims[l + 1];
  c.horizon = w.m;
  c.num_envs = gpg * num_env;
  c.gmis_per_gpu = gpg;
  c.device = ps.device;
  c.gmi_backend = ps.backend;
  // shapes the iteration cannot run (minibatch rows per GMI must tile by 64) are not runnable
  if ((long long)num_env * c.horizon % (64LL * c.minibatches) != 0) return;
  GMI_CUDA_CHECK(cudaSetDevice(ps.device));
  GMI_CUDA_CHECK(cudaDeviceSynchronize());
  size_t free0 = 0, total = 0;
  GMI_CUDA_CHECK(cudaMemGetInfo(&free0, &total));
  std::unique_ptr<Trainer> t;
  try {
    t = std::make_unique<Trainer>(c, nullptr);
  } catch (const Error& e) {
    cudaGetLastError();  // clear a sticky allocation failure
    if (e.code == GMI_ERR_CUDA || e.code == GMI_ERR_INVALID) return;  // does not fit / cannot partition
    throw;
  }
  t->enqueue_iteration(true);  // warm-up (first iteration runs eagerly)
  t->enqueue_iteration(false);  // graph capture
  t->synchronize(nullptr);
  size_t free1 = 0;
  GMI_CUDA_CHECK(cudaMemGetInfo(&free1, &total));
  cudaEvent_t a, b;
  GMI_CUDA_CHECK(cudaEventCreate(&a));
  GMI_CUDA_CHECK(cudaEventCreate(&b));
  GMI_CUDA_CHECK(cudaEventRecord(a, t->stream(-1)));
  for (int i = 0; i < ps.iters; ++i) t->enqueue_iteration(false);
  GMI_CUDA_CHECK(cudaEventRecord(b, t->stream(-1)));
  gmi_ppo_stats_t st;
  t->synchronize(&st);
  float ms = 0.f;
  GMI_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  const double steps = double(st.env_steps) * ps.iters;  // whole GPU
  *runnable = 1;
  *top = steps / (double(ms) / 1e3) / gpg;
  *mem = double(free0 > free1 ? free0 - free1 : 0) / 1e9 / gpg;
}

}  // namespace

}  // namespace gmi

extern "C" {

GMI_API int gmi_gpu_profile(const char* bench, int gmis_per_gpu, int num_env, int device, int backend, int iters,
                            int* runnable, double* top, double* mem) {
  return gmi::guarded([&] {
    if (iters < 1) gmi::invalid("iters must be >= 1");
    gmi::measure(bench, gmis_per_gpu, num_env, {device, backend, iters}, runnable, top, mem);
  });
}

// gmi_probe_fn adapter: user -> int[3] {device, backend, iters}
GMI_API int gmi_gpu_probe(void* user, const char* bench, int gmis_per_gpu, int num_env, int* runnable, double* top,
                          double* mem) {
  const int* s = static_cast<const int*>(user);
  return gmi_gpu_profile(bench, gmis_per_gpu, num_env, s ? s[0] : 0, s ? s[1] : 1, s ? s[2] : 3, runnable, top,
                         mem);
}

}  // extern "C"
