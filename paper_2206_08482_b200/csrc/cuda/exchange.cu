// Cross-GPU gradient exchange fused with Adam over peer memory (the B200 form of the HAR leader
// all-reduce, reduction.hpp:287-299, followed by the update): reduce-scatter -> sharded Adam ->
// all-gather in ONE kernel per minibatch update, no NCCL.
//
// Every rank (one per GPU, num_gpus ranks) owns an exchange window in its HBM -- flags, the
// published gradient (its GMIs' K1 fold), the fp32 master parameters and their bf16 shadow --
// mapped into every peer (CUDA IPC across processes, plain pointers inside one process). Per
// update s (1-based, replay-safe: derived from the device control block):
//   1. signal: rank r publishes ready[r] = s (release, system scope) once its fold is final,
//      and one warp waits until every peer's ready[q] >= s;
//   2. exchange_adam: for its slice of
//      rank r's shard [P r/G, P (r+1)/G) sums the published gradients over NVLink in the fold
//      order of the strategy Alg. 1 selects for the job layout (reduction.hpp:98-106): HAR =
//      the leaders' ring over the ranks' K1 folds; MRR = t rings of one GMI per rank, their
//      results summed into a zero total in ring order (reduction.hpp:255-283); chunk c of every
//      ring starts at member c (:164-212; oracle/ppo_oracle.c fold_gradients). Runs Adam on the shard (Adam
//      moments are sharded: each element's m, v live only on its owner) and stores the new
//      parameter and its bf16 shadow into EVERY rank's window (the all-gather), then stores its
//      (rank, CTA) done flag = s into every rank's window (release; no contended atomics);
//   3. wait: one CTA spins until all G x C done flags in its own window reached s (every CTA of
//      every rank finished writing step s into this rank), so the next minibatch reads final weights.
// No float atomics: every element is summed by exactly one owner in a fixed order, so all ranks
// hold bit-identical parameters, and the arithmetic of the update is adam_kernel's.
#include <cuda_bf16.h>

#include "../host/errors.hpp"
#include "launch.cuh"
#include "ppo.cuh"

namespace gmi::ppo {

namespace {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Flags of a one-rank exchange never leave the GPU: device scope avoids the system-scope
// memory barrier (ERRBAR) a release.sys costs every CTA.
__device__ __forceinline__ void flag_store(unsigned long long* p, unsigned long long v, bool sys) {
  if (sys)
    st_release_sys(p, v);
  else
    st_release_gpu(p, v);
}

__device__ __forceinline__ void spin_until(const unsigned long long* p, unsigned long long target, bool sys) {
  unsigned ns = 32;
  while ((sys ? ld_acquire_sys(p) : ld_acquire_gpu(p)) < target) {
    __nanosleep(ns);
    ns = ns < 1024 ? ns * 2 : ns;
  }
}

__device__ __forceinline__ long long step_id(const ExchangeArgs& a) {
  return a.ctl->adam_step0 + a.step_in_iter + 1;  // 1-based, consecutive over the job
}

// One warp: publish this rank's readiness, then wait for every peer's. The waiting happens
// here, in a single small CTA, and never in the wide exchange kernel: a spinning CTA holds an
// SM slot, and ranks that share a GPU (tests, or several ranks per device) must leave room for
// the peers' persistent GEMMs to finish the gradients being waited for.
__global__ void __launch_bounds__(32) exchange_signal_kernel(const __grid_constant__ ExchangeArgs a) {
  pdl_trigger();
  pdl_wait();  // the fold that produced pub[rank] has completed (device scope)
  const long long s = step_id(a);
  const bool sys = a.G > 1;
  if (threadIdx.x == 0) flag_store(a.ready[a.rank], (unsigned long long)s, sys);  // release: orders the fold
  if (int(threadIdx.x) < a.G) spin_until(a.ready[threadIdx.x], (unsigned long long)s, sys);
  __syncwarp();
}

// FOLD 0: leader ring over the ranks' published folds (HAR, or one rank with one GMI);
// FOLD 1: MRR rings over per-GMI gradients; FOLD 2: one rank, the K1 fold of its t GMIs in the
// MPR ring order (reduction.hpp:164-212) fused in front of Adam -- no separate K1 launch.
template <int FOLD>
__global__ void __launch_bounds__(256) exchange_adam_kernel(const __grid_constant__ ExchangeArgs a) {
  pdl_trigger();
  pdl_wait();  // exchange_signal_kernel completed: every peer's gradient of this step is published
  const long long s = step_id(a);
  const long long st = s - 1;  // completed updates before this one (bias-correction index)
  const float bc1 = a.bc[2 * st], bc2 = a.bc[2 * st + 1];
  const float ob1 = __fsub_rn(1.0f, a.b1), ob2 = __fsub_rn(1.0f, a.b2);
  float* __restrict__ mom = a.m;
  float* __restrict__ vel = a.v;
  const float* __restrict__ own = a.params[a.rank];
  // Each thread owns up to kX elements per pass and issues all their loads before any store
  // (kept small and not unrolled over the ranks: the kernel stays inside the instruction cache).
  constexpr int kX = 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = a.lo + (long long)blockIdx.x * blockDim.x + threadIdx.x; base < a.hi; base += kX * stride) {
    float gsum[kX], m0[kX], v0[kX], p0[kX];
#pragma unroll
    for (int u = 0; u < kX; ++u) {
      const long long i = base + u * stride;
      gsum[u] = m0[u] = v0[u] = p0[u] = 0.f;
      if (i >= a.hi) continue;
      // chunk cg = the ring chunk holding element i (chunk c = [P c / G, P (c + 1) / G),
      // reduction.hpp:164-166); every ring fold starts at member cg
      int cg = 0;
      while (cg + 1 < a.G && i >= a.chunk0[cg + 1]) ++cg;
      float acc = 0.f;
      if constexpr (FOLD == 2) {  // one rank: MPR ring over its t GMI gradients, chunk c starts at member c
        int c = 0;
        while (c + 1 < a.t && i >= a.chunk0_t[c + 1]) ++c;
#pragma unroll 1
        for (int j = 0; j < a.t; ++j) {
          int r = c + j;
          r -= r >= a.t ? a.t : 0;
          const float x = a.gpub[0][r][i];
          acc = j == 0 ? x : __fadd_rn(x, acc);
        }
      } else if constexpr (FOLD == 0) {  // HAR leader ring (or one rank): the ranks' K1 folds in ring order
#pragma unroll 1
        for (int j = 0; j < a.G; ++j) {
          int q = cg + j;
          q -= q >= a.G ? a.G : 0;
          const float x = __ldcg(a.pub[q] + i);  // peer memory: L2 of the owner, never a stale L1 line
          acc = j == 0 ? x : __fadd_rn(x, acc);
        }
      } else {  // MRR: ring r = GMI r of ranks r, r+1, ...; ring results into a zero total in ring order
#pragma unroll 1
        for (int r = 0; r < a.t; ++r) {
          float ring = 0.f;
#pragma unroll 1
          for (int j = 0; j < a.G; ++j) {
            int q = r + cg + j;
            q %= a.G;
            const float x = __ldcg(a.gpub[q][r] + i);
            ring = j == 0 ? x : __fadd_rn(x, ring);
          }
          acc = __fadd_rn(acc, ring);
        }
      }
      gsum[u] = acc;
      m0[u] = mom[i];
      v0[u] = vel[i];
      p0[u] = own[i];
    }
#pragma unroll
    for (int u = 0; u < kX; ++u) {
      const long long i = base + u * stride;
      if (i >= a.hi) break;
      const float g = __fmul_rn(gsum[u], a.inv_n);
      const float m = __fadd_rn(__fmul_rn(a.b1, m0[u]), __fmul_rn(ob1, g));
      const float v = __fadd_rn(__fmul_rn(a.b2, v0[u]), __fmul_rn(__fmul_rn(ob2, g), g));
      mom[i] = m;
      vel[i] = v;
      const float mh = __fdiv_rn(m, bc1), vh = __fdiv_rn(v, bc2);
      const float p = __fsub_rn(p0[u], __fmul_rn(a.lr, __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), a.eps))));
      const __nv_bfloat16 sh = __float2bfloat16_rn(p);
#pragma unroll 1
      for (int q = 0; q < a.G; ++q) {  // all-gather: the owner writes every replica
        a.params[q][i] = p;
        a.shadow[q][i] = sh;
      }
    }
  }
  if (a.G == 1) return;  // one rank: stream order is the only consumer
  __syncthreads();  // the CTA's stores happen-before the releases below (bar.sync + release cumulativity)
  // one flag per (rank, CTA) in every destination's window -- plain release stores, no
  // contended atomics on one counter
  if (int(threadIdx.x) < a.G)
    flag_store(a.done[threadIdx.x] + a.rank * kMaxXchgCtas + blockIdx.x, (unsigned long long)s, a.G > 1);
}

// One CTA: wait until every (source rank, CTA) flag in this rank's window reached step s.
__global__ void __launch_bounds__(256) exchange_wait_kernel(const __grid_constant__ ExchangeArgs a) {
  pdl_trigger();
  pdl_wait();
  const unsigned long long s = (unsigned long long)step_id(a);
  for (int f = threadIdx.x; f < a.G * a.ctas; f += blockDim.x) {
    const int q = f / a.ctas, c = f - q * a.ctas;
    spin_until(a.done[a.rank] + q * kMaxXchgCtas + c, s, a.G > 1);
  }
  __syncthreads();
}

// ------------------------------------------------------------------ cross-GPU experience link
// AsyncDecoupled across GPUs (cfg.decoupled = 2): one thread waits until the flag(s) in this
// GPU's link window reach the next target of a device-resident counter (graph-replay safe:
// target = ++ctr + add), or signals a peer's flag the same way after a system-scope fence
// (the copies enqueued before it on the stream have completed). A wait that does not complete
// within 60 s traps, so a dead peer surfaces as a kernel error instead of a hung GPU.
__global__ void link_wait_kernel(const unsigned long long* f1, const unsigned long long* f2, unsigned long long* ctr,
                                 unsigned long long add) {
  if (threadIdx.x != 0) return;
  const unsigned long long target = *ctr + 1 + add;
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned ns = 64;
  while (ld_acquire_sys(f1) < target || (f2 != nullptr && ld_acquire_sys(f2) < target)) {
    __nanosleep(ns);
    ns = ns < 2048 ? ns * 2 : ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 60000000000ull) asm volatile("trap;");
  }
  *ctr += 1;
}

__global__ void link_signal_kernel(unsigned long long* flag, unsigned long long* ctr, unsigned long long add) {
  if (threadIdx.x != 0) return;
  const unsigned long long v = *ctr + 1 + add;
  *ctr += 1;
  __threadfence_system();
  st_release_sys(flag, v);
}

}  // namespace

void launch_link_wait(const unsigned long long* f1, const unsigned long long* f2, unsigned long long* ctr,
                      unsigned long long add, cudaStream_t s) {
  link_wait_kernel<<<1, 32, 0, s>>>(f1, f2, ctr, add);
  GMI_CUDA_CHECK(cudaGetLastError());
}

void launch_link_signal(unsigned long long* flag, unsigned long long* ctr, unsigned long long add, cudaStream_t s) {
  link_signal_kernel<<<1, 32, 0, s>>>(flag, ctr, add);
  GMI_CUDA_CHECK(cudaGetLastError());
}

void launch_exchange_adam(const ExchangeArgs& a, cudaStream_t s) {
  if (a.G < 1 || a.G > kMaxRanks) invalid("exchange: 1..8 ranks");
  if (a.ctas < 1 || a.ctas > kMaxXchgCtas) invalid("exchange: 1..1184 CTAs");
  if (a.G == 1) {  // one rank: no peers to publish to or wait for; the GMI fold is fused in
    if (a.t > 1)
      launch_pdl(exchange_adam_kernel<2>, dim3(a.ctas), dim3(256), 0, s, a);
    else
      launch_pdl(exchange_adam_kernel<0>, dim3(a.ctas), dim3(256), 0, s, a);
    return;
  }
  launch_pdl(exchange_signal_kernel, dim3(1), dim3(32), 0, s, a);
  if (a.mrr)
    launch_pdl(exchange_adam_kernel<1>, dim3(a.ctas), dim3(256), 0, s, a);
  else
    launch_pdl(exchange_adam_kernel<0>, dim3(a.ctas), dim3(256), 0, s, a);
  launch_pdl(exchange_wait_kernel, dim3(1), dim3(256), 0, s, a);
}

}  // namespace gmi::ppo
