// Warp-level helpers shared by the PPO kernels (ppo_kernels.cu, ppo_update.cu).
#pragma once

#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>

namespace gmi::ppo {

constexpr float kLog2PiHalf = 0.91893853320467274f;  // 0.5 * log(2 pi)

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Reduce NV per-lane partial vectors across the warp so that lane l ends with the full sum
// of entry (l % NV): butterfly for offsets >= NV, then recursive halving (NV - 1 shuffles).
template <int NV>
__device__ __forceinline__ float warp_reduce_transpose(float (&v)[NV]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o >= NV; o >>= 1)
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
#pragma unroll
  for (int o = NV / 2; o >= 1; o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const float send = upper ? v[i] : v[i + o];
      const float keep = upper ? v[i + o] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0];
}

__device__ __forceinline__ float elu_grad(float h) { return h > 0.f ? 1.f : h + 1.f; }

// sin of an env state coordinate in the dynamics' coupling term. States stay within a few
// units of 0, where the SFU sine has absolute error ~5e-7; the term is scaled by
// DT * COUPLE = 5e-3 before it reaches the state, far below the bf16 observation rounding.
// Shared by the fused rollout and act_env_kernel so both device paths agree bit-for-bit.
__device__ __forceinline__ float env_sin(float x) { return __sinf(x); }

__device__ __forceinline__ float2 ld_bf16x2(const __nv_bfloat16* p) {
  const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(p);
  return make_float2(__bfloat162float(b.x), __bfloat162float(b.y));
}

__device__ __forceinline__ void st_bf16x2(__nv_bfloat16* p, float a, float b) {
  *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(a, b);
}

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
    f[2 * i] = __bfloat162float(b.x);
    f[2 * i + 1] = __bfloat162float(b.y);
  }
}

inline int grid_for(long long work, int block, int cap) {
  return int(std::max<long long>(1, std::min<long long>((work + block - 1) / block, cap)));
}

}  // namespace gmi::ppo
