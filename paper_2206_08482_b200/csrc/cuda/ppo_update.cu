// PPO update-phase kernels (K6 head + clipped-surrogate loss + head backward, bias-gradient
// column sums, fixed-order gradient assembly). The weight gradients of every layer,
// including the heads, are tcgen05 GEMMs (gemm.cuh); these kernels are HBM-bound.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "../host/errors.hpp"
#include "ppo.cuh"
#include "ppo_common.cuh"

namespace gmi::ppo {

namespace {

// ------------------------------------------------------------------ K6 head + PPO loss
// One warp per minibatch row (8 rows per warp, 64 per block). Lane owns hidden units
// k = 2*lane + 64 j (+1). Per row: mu and v (transpose-reduced dot products against the
// smem-staged head weights), Gaussian log-prob, ratio, clipped surrogate and value loss,
// dL/dmu, dL/dv (also written bf16 into G_pi / G_v for the head weight-gradient GEMM),
// dL/dlog_std, and the head backward dPre_L = (g W) * elu'(H_L) for both nets (bf16).
// Traffic per row: read 2 hp bf16 (H_pi, H_v) + A+4 fp32, write 2 hp bf16 + (A+1) bf16.
template <int NV>
__global__ void __launch_bounds__(256) head_loss_kernel(const HeadLossArgs a) {
  extern __shared__ float sm[];
  __shared__ float red_s[8][69];
  const int A = a.A, hp = a.hp;
  float* w_s = sm;            // [A][hp]
  float* wv_s = sm + A * hp;  // [hp]
  for (int i = threadIdx.x; i < A * hp; i += blockDim.x) w_s[i] = a.w_mu[i];
  for (int i = threadIdx.x; i < hp; i += blockDim.x) wv_s[i] = a.w_v[i];
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float invB = 1.0f / float(a.B);
  const float ls = lane < A ? a.log_std[lane] : 0.f;
  const float sig = expf(ls);
  const float bmu = lane < A ? a.b_mu[lane] : 0.f;
  const float bv = a.b_v[0];
  float acc_db = 0.f, acc_ls = 0.f, acc_dbv = 0.f, st0 = 0.f, st1 = 0.f, st2 = 0.f, st3 = 0.f;
  constexpr int kRowsPerWarp = kHeadRowsPerBlock / 8;
  constexpr int kJ = kMaxHeadIn / 64;
  const int rbeg = blockIdx.x * kHeadRowsPerBlock + warp * kRowsPerWarp;

  for (int rr = 0; rr < kRowsPerWarp; ++rr) {
    const int r = rbeg + rr;
    if (r >= a.B) break;  // warp-uniform
    float2 h[kJ], hv[kJ];
    float part[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) part[i] = 0.f;
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int k = 2 * lane + 64 * j;
      if (k < hp) {
        h[j] = ld_bf16x2(a.Hpi + (long long)r * hp + k);
        hv[j] = ld_bf16x2(a.Hv + (long long)r * hp + k);
#pragma unroll
        for (int i = 0; i < NV - 1; ++i)
          if (i < A) {
            const float2 w = *reinterpret_cast<const float2*>(w_s + i * hp + k);
            part[i] += h[j].x * w.x + h[j].y * w.y;
          }
        const float2 wv = *reinterpret_cast<const float2*>(wv_s + k);
        part[NV - 1] += hv[j].x * wv.x + hv[j].y * wv.y;
      }
    }
    const float red = warp_reduce_transpose<NV>(part);
    const float mu = red + bmu;  // lanes < A
    const float v = __shfl_sync(0xffffffffu, red, NV - 1) + bv;
    float z = 0.f, term = 0.f;
    if (lane < A) {
      z = (a.act[(long long)r * A + lane] - mu) / sig;
      term = -0.5f * z * z - ls - kLog2PiHalf;
    }
    const float lp = warp_sum(term);
    const float oldlp = a.oldlp[r], adv = a.adv[r];
    const float ratio = expf(lp - oldlp);
    const float s1 = ratio * adv;
    const float rc = fminf(fmaxf(ratio, 1.f - a.clip), 1.f + a.clip);
    const float s2 = rc * adv;
    const bool take1 = s1 <= s2;
    const float glp = take1 ? -s1 * invB : 0.f;
    const float verr = v - a.ret[r];
    const float gv = a.vf_coef * verr * invB;
    float gmu = 0.f;
    if (lane < A) {
      gmu = glp * z / sig;
      acc_db += gmu;
      acc_ls += glp * (z * z - 1.f) - a.ent_coef * invB;
      a.Gpi[(long long)r * kHeadG + lane] = __float2bfloat16_rn(gmu);
    }
    if (lane == 0) {
      a.Gv[(long long)r * kHeadG] = __float2bfloat16_rn(gv);
      acc_dbv += gv;
      st0 += -(take1 ? s1 : s2);
      st1 += 0.5f * a.vf_coef * verr * verr;
      st2 += oldlp - lp;
      st3 += (ratio < 1.f - a.clip || ratio > 1.f + a.clip) ? 1.f : 0.f;
    }
    float g_all[NV - 1];
#pragma unroll
    for (int i = 0; i < NV - 1; ++i) g_all[i] = __shfl_sync(0xffffffffu, gmu, i);
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int k = 2 * lane + 64 * j;
      if (k < hp) {
        float d0 = 0.f, d1 = 0.f;
#pragma unroll
        for (int i = 0; i < NV - 1; ++i)
          if (i < A) {
            const float2 w = *reinterpret_cast<const float2*>(w_s + i * hp + k);
            d0 += g_all[i] * w.x;
            d1 += g_all[i] * w.y;
          }
        st_bf16x2(a.Dpi + (long long)r * hp + k, d0 * elu_grad(h[j].x), d1 * elu_grad(h[j].y));
        const float2 wv = *reinterpret_cast<const float2*>(wv_s + k);
        st_bf16x2(a.Dv + (long long)r * hp + k, (gv * wv.x) * elu_grad(hv[j].x), (gv * wv.y) * elu_grad(hv[j].y));
      }
    }
  }
  red_s[warp][lane] = lane < A ? acc_db : 0.f;
  red_s[warp][32 + lane] = lane < A ? acc_ls : 0.f;
  if (lane == 0) {
    red_s[warp][64] = acc_dbv;
    red_s[warp][65] = st0;
    red_s[warp][66] = st1;
    red_s[warp][67] = st2;
    red_s[warp][68] = st3;
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < 2 * A + 5) {
    int col;
    if (t < A) col = t;                       // db_mu
    else if (t == A) col = 64;                // db_v
    else if (t < 2 * A + 1) col = 32 + (t - A - 1);  // dlog_std
    else col = 65 + (t - 2 * A - 1);          // statistics
    float s = 0.f;
    for (int w = 0; w < 8; ++w) s += red_s[w][col];
    a.partial[(long long)blockIdx.x * head_partial_stride(A) + t] = s;
  }
}

// ------------------------------------------------------------------ bias-gradient column sums
// Block = 256 rows x all columns of one problem; thread = 2 adjacent columns with 8
// independent row accumulators combined in a fixed tree order (deterministic).
constexpr int kColsumRows = 256;
struct ColsumArgs {
  const __nv_bfloat16* D[16];
  float* out[16];
  int width[16];
};
__global__ void __launch_bounds__(128) colsum_kernel(const ColsumArgs a, int rows) {
  const int p = blockIdx.y;
  const int w = a.width[p];
  const int r0 = blockIdx.x * kColsumRows;
  const int r1 = min(rows, r0 + kColsumRows);
  const __nv_bfloat16* D = a.D[p];
  for (int c = 2 * threadIdx.x; c < w; c += 2 * blockDim.x) {
    float sx[8] = {}, sy[8] = {};
    int r = r0;
    for (; r + 8 <= r1; r += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float2 v = ld_bf16x2(D + (long long)(r + u) * w + c);
        sx[u] += v.x;
        sy[u] += v.y;
      }
    }
    for (; r < r1; ++r) {
      const float2 v = ld_bf16x2(D + (long long)r * w + c);
      sx[0] += v.x;
      sy[0] += v.y;
    }
    const float tx = ((sx[0] + sx[1]) + (sx[2] + sx[3])) + ((sx[4] + sx[5]) + (sx[6] + sx[7]));
    const float ty = ((sy[0] + sy[1]) + (sy[2] + sy[3])) + ((sy[4] + sy[5]) + (sy[6] + sy[7]));
    a.out[p][(long long)blockIdx.x * w + c] = tx;
    a.out[p][(long long)blockIdx.x * w + c + 1] = ty;
  }
}

// ------------------------------------------------------------------ gradient assembly
constexpr int kMaxSegments = 64;
struct SegmentTable {
  Segment s[kMaxSegments];
};
__global__ void __launch_bounds__(256) segments_kernel(const __grid_constant__ SegmentTable t) {
  const Segment& sg = t.s[blockIdx.y];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < sg.len; i += gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < sg.nparts; ++p) acc += sg.src[(long long)p * sg.stride + i];
    sg.dst[i] = acc;
  }
}

}  // namespace

int head_loss_blocks(int B) { return (B + kHeadRowsPerBlock - 1) / kHeadRowsPerBlock; }

void launch_head_loss(const HeadLossArgs& a, cudaStream_t s) {
  if (a.A > kMaxAct) invalid("act_dim > 31 unsupported by the head kernel");
  if (a.hp > kMaxHeadIn) invalid("last hidden width > 512 unsupported by the head kernel");
  const int blocks = head_loss_blocks(a.B);
  const size_t smem = (size_t(a.A) + 1) * a.hp * 4;
  auto go = [&](auto kern) {
    if (smem > 40 * 1024)
      GMI_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<blocks, 256, smem, s>>>(a);
  };
  if (a.A <= 7)
    go(head_loss_kernel<8>);
  else if (a.A <= 15)
    go(head_loss_kernel<16>);
  else
    go(head_loss_kernel<32>);
  GMI_CUDA_CHECK(cudaGetLastError());
}

int colsum_blocks(int rows) { return (rows + kColsumRows - 1) / kColsumRows; }

void launch_colsum(const __nv_bfloat16* const* D, const int* widths, float* const* partial, int np, int rows,
                   cudaStream_t s) {
  if (np > 16) invalid("too many column-sum problems");
  ColsumArgs a{};
  for (int i = 0; i < np; ++i) {
    if (widths[i] % 2) invalid("column-sum width must be even");
    a.D[i] = D[i];
    a.out[i] = partial[i];
    a.width[i] = widths[i];
  }
  colsum_kernel<<<dim3(colsum_blocks(rows), np), 128, 0, s>>>(a, rows);
  GMI_CUDA_CHECK(cudaGetLastError());
}

void launch_segments(const Segment* segs, int n, cudaStream_t s) {
  for (int base = 0; base < n; base += kMaxSegments) {
    SegmentTable t{};
    const int m = std::min(kMaxSegments, n - base);
    int maxlen = 1;
    for (int i = 0; i < m; ++i) {
      t.s[i] = segs[base + i];
      maxlen = std::max(maxlen, t.s[i].len);
    }
    segments_kernel<<<dim3(grid_for(maxlen, 256, 1024), m), 256, 0, s>>>(t);
    GMI_CUDA_CHECK(cudaGetLastError());
  }
}

}  // namespace gmi::ppo
