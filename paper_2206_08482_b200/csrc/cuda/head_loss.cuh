// Per-row PPO head loss shared by the fused head kernels (head_fused.cu, train_fwd.cu).
// Numerics follow head_loss_kernel (ppo_update.cu) and oracle/ppo_oracle.c: Gaussian
// log-prob summed in action order, clipped surrogate, value loss 0.5 (v - R)^2 vf_coef.
//
// Thread = minibatch row (its TMEM lane); r[] holds the row's head accumulator columns
// (mu or v, bias not yet added). Per-action sums over rows (head-bias and log-std gradients):
// for A <= 8 each thread keeps running sums in registers (head_loss_flush reduces them at the
// end); for wider action spaces they are reduced per warp every tile and added by lane 0 into
// the warp's shared-memory record, so no large per-action register arrays persist across
// tiles (A up to 31 without spills). Both orders are fixed, so results are deterministic.
#pragma once

#include <cuda_bf16.h>

#include <cstdint>

#include "ppo_common.cuh"

namespace gmi::ppo {

// cst (shared): [0, 32) log_std, [32, 64) exp(log_std), [64, 96) head bias of this net,
// [96, 128) 1 / exp(log_std).
// lacc (shared, this warp): [i] sum of dL/dmu_i (or dL/dv), [32 + i] sum of dL/dlog_std_i.
// st: running loss statistics of this thread's rows {policy loss, value loss, kl, clipped}.
// G row: bf16 dL/dout into the SW128 K-major tile row `grow_s` (16-byte units swizzled by row & 7);
// columns [n_out, nh) are written as zeros.
template <int MAXA>
constexpr bool kLossRegAcc = MAXA <= 8;
// actions prefetched into registers before the accumulator wait (one round trip for the row's
// actions instead of a dependent load per action between the G stores): A <= 24
template <int MAXA>
constexpr bool kLossPre = MAXA <= 24;
template <int MAXA>
constexpr int kActRegs = kLossPre<MAXA> ? MAXA : 1;

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int MAXA>
__device__ __forceinline__ void head_row_loss(int net, const uint32_t (&r)[32], const float* cst, int nout, int nh,
                                              bool valid, const float* act_row, float (&act_r)[kActRegs<MAXA>],
                                              float oldlp, float adv, float ret, float clip, float vf_coef,
                                              float ent_coef, float invB, uint8_t* grow_s, int row, float* lacc,
                                              float (&st)[4], float (&sg)[kLossRegAcc<MAXA> ? MAXA : 1],
                                              float (&sl)[kLossRegAcc<MAXA> ? MAXA : 1]) {
  constexpr bool kPre = kLossPre<MAXA>;  // actions prefetched into registers before the accumulator wait
  constexpr int kGk = kPre ? (MAXA + 7) / 8 * 8 : 1;  // packed G row: 16-byte units of 8 bf16
  const int lane = threadIdx.x & 31;
  auto put_g = [&](int col, float v) {
    *reinterpret_cast<__nv_bfloat16*>(grow_s + ((((col >> 3) ^ (row & 7))) << 4) + (col & 7) * 2) =
        __float2bfloat16_rn(v);
  };
  auto zero_row = [&](int from_unit) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (u >= from_unit && u * 8 < nh) *reinterpret_cast<uint4*>(grow_s + ((u ^ (row & 7)) << 4)) = make_uint4(0u, 0u, 0u, 0u);
  };
  // z_i = (a_i - mu_i) / sigma_i, as a multiply by 1 / sigma_i (cst[96 + i]); with prefetched
  // actions the registers are reused for z
  auto zval = [&](int i) {
    const float mu = __uint_as_float(r[i]) + cst[64 + i];
    return ((kPre ? act_r[kPre ? i : 0] : act_row[i]) - mu) * cst[96 + i];
  };
  if (net == 0) {
    float lp = 0.f;
#pragma unroll
    for (int i = 0; i < MAXA; ++i)
      if (i < nout && valid) {
        const float z = zval(i);
        if constexpr (kPre) act_r[i] = z;
        lp += -0.5f * z * z - cst[i] - kLog2PiHalf;
      }
    float glp = 0.f;
    if (valid) {
      const float ratio = expf(lp - oldlp);
      const float s1 = ratio * adv;
      const float rc = fminf(fmaxf(ratio, 1.f - clip), 1.f + clip);
      const float s2 = rc * adv;
      const bool take1 = s1 <= s2;
      glp = take1 ? -s1 * invB : 0.f;
      st[0] += -(take1 ? s1 : s2);
      st[2] += oldlp - lp;
      st[3] += (ratio < 1.f - clip || ratio > 1.f + clip) ? 1.f : 0.f;
    }
    if constexpr (!kPre) zero_row(0);
    float gk[kGk];  // small action spaces: the G row is packed and stored as 16-byte units
#pragma unroll
    for (int i = 0; i < kGk; ++i) gk[i] = 0.f;
#pragma unroll
    for (int i = 0; i < MAXA; ++i)
      if (i < nout) {
        float g = 0.f, gl = 0.f;
        if (valid) {
          const float z = kPre ? act_r[kPre ? i : 0] : zval(i);
          g = glp * z * cst[96 + i];
          gl = glp * (z * z - 1.f) - ent_coef * invB;
        }
        if constexpr (kPre) gk[i] = g;
        else put_g(i, g);
        if constexpr (kLossRegAcc<MAXA>) {
          sg[i] += g;
          sl[i] += gl;
        } else if constexpr (!kPre) {
          g = warp_sum(g);
          gl = warp_sum(gl);
          if (lane == 0) {
            lacc[i] += g;
            lacc[32 + i] += gl;
          }
        }
      }
    if constexpr (kPre) {
      constexpr int kUnits = kGk / 8 < 2 ? 2 : kGk / 8;  // >= the 16 columns of the smallest head
      auto gv = [&](int k) { return k < kGk ? gk[k] : 0.f; };
#pragma unroll
      for (int u = 0; u < kUnits; ++u)
        *reinterpret_cast<uint4*>(grow_s + ((u ^ (row & 7)) << 4)) =
            make_uint4(pack2(gv(8 * u), gv(8 * u + 1)), pack2(gv(8 * u + 2), gv(8 * u + 3)),
                       pack2(gv(8 * u + 4), gv(8 * u + 5)), pack2(gv(8 * u + 6), gv(8 * u + 7)));
      zero_row(kUnits);
      if constexpr (!kLossRegAcc<MAXA>) {
        // per-action sums over the warp's rows (head-bias and log-std gradients), 8 actions at a
        // time: 8 independent reductions per shuffle step (butterfly over lanes 16 / 8, then
        // recursive halving) leave action c * 8 + l's sum on lane l, which adds it to the record
        // -- instead of a dependent 5-shuffle chain and a serial shared-memory update per action
#pragma unroll
        for (int c = 0; c < (MAXA + 7) / 8; ++c) {
          float v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = c * 8 + u < nout ? gk[(c * 8 + u) % kGk] : 0.f;
          float sum = warp_reduce_transpose<8>(v);
          if (lane < 8 && c * 8 + lane < nout) lacc[c * 8 + lane] += sum;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int i = c * 8 + u;
            const float z = act_r[i % kActRegs<MAXA>];
            v[u] = i < nout ? (valid ? glp * (z * z - 1.f) - ent_coef * invB : 0.f) : 0.f;
          }
          sum = warp_reduce_transpose<8>(v);
          if (lane < 8 && c * 8 + lane < nout) lacc[32 + c * 8 + lane] += sum;
        }
      }
    }
  } else {
    zero_row(0);
    float g = 0.f;
    if (valid) {
      const float v = __uint_as_float(r[0]) + cst[64];
      const float verr = v - ret;
      g = vf_coef * verr * invB;
      st[1] += 0.5f * vf_coef * verr * verr;
    }
    put_g(0, g);
    if constexpr (kLossRegAcc<MAXA>) {
      sg[0] += g;
    } else {
      g = warp_sum(g);
      if (lane == 0) lacc[0] += g;
    }
  }
}

// End of the CTA's tiles: register-held per-action sums and the loss statistics into the warp's
// shared-memory record ([0, 64) per-action sums, [64, 68) statistics).
template <int MAXA>
__device__ __forceinline__ void head_loss_flush(int nout, float* lacc, const float (&st)[4],
                                                const float (&sg)[kLossRegAcc<MAXA> ? MAXA : 1],
                                                const float (&sl)[kLossRegAcc<MAXA> ? MAXA : 1]) {
  const int lane = threadIdx.x & 31;
  if constexpr (kLossRegAcc<MAXA>) {
#pragma unroll
    for (int i = 0; i < MAXA; ++i)
      if (i < nout) {
        const float a = warp_sum(sg[i]), b = warp_sum(sl[i]);
        if (lane == 0) {
          lacc[i] += a;
          lacc[32 + i] += b;
        }
      }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float x = warp_sum(st[k]);
    if (lane == 0) lacc[64 + k] = x;
  }
}

}  // namespace gmi::ppo
