// PPO update-phase kernels: K6 clipped-surrogate / value loss (elementwise over the
// head-GEMM outputs), bias-gradient column sums, and the fixed-order gradient assembly.
// Every matrix product of the update (hidden layers and both heads, forward, input- and
// weight-gradients) is a tcgen05 GEMM (gemm.cuh); these kernels are HBM/L2-bound.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "../host/errors.hpp"
#include "launch.cuh"
#include "ppo.cuh"
#include "ppo_common.cuh"

namespace gmi::ppo {

namespace {

// ------------------------------------------------------------------ K6 loss + head gradients
// Thread per minibatch row. Inputs: mu / v from the head GEMMs (+ bias), stored action,
// old log-prob, normalised advantage, return. Outputs: dL/dmu and dL/dv as bf16 rows of
// G_pi / G_v (operands of the head input- and weight-gradient GEMMs) and one block partial
// of db_mu[A], db_v, dlog_std[A] and the loss statistics. Sums over actions run in action
// order, like the oracle. Traffic per row: (2A + 5) x 4 B read, 2 (A + 1) B written.
template <int MAXA>
__global__ void __launch_bounds__(256) head_loss_kernel(const HeadLossArgs a) {
  __shared__ float red_s[8][2 * kMaxAct + 5];
  pdl_trigger();
  pdl_wait();
  const int A = a.A;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float invB = 1.0f / float(a.B);
  float gmu[MAXA], gls[MAXA];
  float gv = 0.f, st0 = 0.f, st1 = 0.f, st2 = 0.f, st3 = 0.f;
#pragma unroll
  for (int i = 0; i < MAXA; ++i) gmu[i] = gls[i] = 0.f;
  if (r < a.B) {
    float mu[MAXA], z[MAXA], ls[MAXA], sig[MAXA];
    float lp = 0.f;
#pragma unroll
    for (int i = 0; i < MAXA; ++i)
      if (i < A) {
        mu[i] = a.mu[(long long)r * kHeadG + i] + a.b_mu[i];
        ls[i] = a.log_std[i];
        sig[i] = expf(ls[i]);
        z[i] = (a.act[(long long)r * A + i] - mu[i]) / sig[i];
        lp += -0.5f * z[i] * z[i] - ls[i] - kLog2PiHalf;
      }
    const float v = a.v[(long long)r * kHeadG] + a.b_v[0];
    const float oldlp = a.oldlp[r], adv = a.adv[r];
    const float ratio = expf(lp - oldlp);
    const float s1 = ratio * adv;
    const float rc = fminf(fmaxf(ratio, 1.f - a.clip), 1.f + a.clip);
    const float s2 = rc * adv;
    const bool take1 = s1 <= s2;
    const float glp = take1 ? -s1 * invB : 0.f;
    const float verr = v - a.ret[r];
    gv = a.vf_coef * verr * invB;
    __nv_bfloat16* grow = a.Gpi + (long long)r * kHeadG;
#pragma unroll
    for (int i = 0; i < MAXA; ++i)
      if (i < A) {
        gmu[i] = glp * z[i] / sig[i];
        gls[i] = glp * (z[i] * z[i] - 1.f) - a.ent_coef * invB;
        grow[i] = __float2bfloat16_rn(gmu[i]);
      }
    a.Gv[(long long)r * kHeadG] = __float2bfloat16_rn(gv);
    st0 = -(take1 ? s1 : s2);
    st1 = 0.5f * a.vf_coef * verr * verr;
    st2 = oldlp - lp;
    st3 = (ratio < 1.f - a.clip || ratio > 1.f + a.clip) ? 1.f : 0.f;
  }
  // block partial: warp butterflies, then warps in order (deterministic)
  auto put = [&](int col, float x) {
    x = warp_sum(x);
    if (lane == 0) red_s[warp][col] = x;
  };
#pragma unroll
  for (int i = 0; i < MAXA; ++i)
    if (i < A) {
      put(i, gmu[i]);
      put(A + 1 + i, gls[i]);
    }
  put(A, gv);
  put(2 * A + 1, st0);
  put(2 * A + 2, st1);
  put(2 * A + 3, st2);
  put(2 * A + 4, st3);
  __syncthreads();
  const int t = threadIdx.x;
  if (t < head_partial_stride(A)) {
    float s = 0.f;
    for (int w = 0; w < 8; ++w) s += red_s[w][t];
    a.partial[(long long)blockIdx.x * head_partial_stride(A) + t] = s;
  }
}

// ------------------------------------------------------------------ bias-gradient column sums
// Block = 128 rows of one problem; 16-byte loads (8 columns per thread), w/8 threads per row,
// 256/(w/8) row lanes; row lanes combined through shared memory in a fixed order.
constexpr int kColsumRows = 128;
struct ColsumArgs {
  const __nv_bfloat16* D[16];
  float* out[16];
  int width[16];
};
__global__ void __launch_bounds__(256) colsum_kernel(const ColsumArgs a, int rows) {
  __shared__ float part_s[2048];  // [row lanes][w]; row lanes * w <= 2048
  pdl_trigger();
  pdl_wait();
  const int p = blockIdx.y;
  const int w = a.width[p];
  const int tpr = w / 8;
  const int lanes = 256 / tpr;
  const int t = threadIdx.x;
  const int rl = t / tpr, c = (t % tpr) * 8;
  const __nv_bfloat16* D = a.D[p];
  const int r0 = blockIdx.x * kColsumRows;
  const int r1 = min(rows, r0 + kColsumRows);
  float s[8] = {};
  if (rl < lanes) {
    for (int r = r0 + rl; r < r1; r += lanes) {
      float f[8];
      load8(D + (long long)r * w + c, f);
#pragma unroll
      for (int j = 0; j < 8; ++j) s[j] += f[j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) part_s[rl * w + c + j] = s[j];
  }
  __syncthreads();
  for (int j = t; j < w; j += blockDim.x) {
    float tot = 0.f;
    for (int l = 0; l < lanes; ++l) tot += part_s[l * w + j];
    a.out[p][(long long)blockIdx.x * w + j] = tot;
  }
}

// ------------------------------------------------------------------ gradient assembly
// dst[i] = sum_p src[p*stride + i]. Block = 128 consecutive elements x 256 threads, summed in a
// fixed order (deterministic, the same for every launch):
//  * vector path (length / stride / pointers 16-byte multiples): one float4 per lane, warp w sums
//    the contiguous part range [w*np/8, (w+1)*np/8) in part order with 4 loads in flight, then the
//    8 warp sums are added in warp order;
//  * lane path (short or unaligned segments: head-bias, log-std and loss-statistic partials, with
//    up to one part per CTA of the head kernel): the block's threads are (group g, element e) with
//    G = 256 / pow2(len) groups; group g sums parts g, g + G, g + 2G, ... (4 loads in flight), then
//    the groups are added in group order. Every part load of the block is in flight at once, where
//    a thread per element walking all parts serially took a dependent round trip per part.
constexpr int kMaxSegments = 64;
constexpr int kSegElems = 128;
// quad path: 16-byte-aligned segments with at most kQuadParts parts (the split-K weight and
// bias-gradient slabs): thread = 4 consecutive elements, all parts loaded before they are summed
// in part order in registers (one round trip, no cross-warp reduction), 1024 elements per block
constexpr int kQuadParts = 16;
constexpr int kQuadElems = 1024;
__host__ __device__ inline bool seg_quad(const Segment& sg) {
  return sg.nparts <= kQuadParts && ((sg.len | (int)(sg.stride & 3)) & 3) == 0 &&
         ((reinterpret_cast<uintptr_t>(sg.src) | reinterpret_cast<uintptr_t>(sg.dst)) & 15) == 0;
}
// Adam on one element, same arithmetic as adam_kernel (bit-identical)
__device__ __forceinline__ void adam_elem(const SegAdam& a, long long i, float gs, float bc1, float bc2) {
  const float ob1 = __fsub_rn(1.0f, a.b1), ob2 = __fsub_rn(1.0f, a.b2);
  const float g = __fmul_rn(gs, a.inv_n);
  const float m = __fadd_rn(__fmul_rn(a.b1, a.m[i]), __fmul_rn(ob1, g));
  const float v = __fadd_rn(__fmul_rn(a.b2, a.v[i]), __fmul_rn(__fmul_rn(ob2, g), g));
  a.m[i] = m;
  a.v[i] = v;
  const float mh = __fdiv_rn(m, bc1), vh = __fdiv_rn(v, bc2);
  const float p = __fsub_rn(a.p[i], __fmul_rn(a.lr, __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), a.eps))));
  a.p[i] = p;
  a.shadow[i] = __float2bfloat16_rn(p);
}
struct SegmentTable {
  Segment s[kMaxSegments];
  int first_block[kMaxSegments + 1];  // prefix of blocks per segment
  int nseg;
  int has_adam;
  SegAdam adam;
};
// kAdam: the fused-Adam variant. 4 blocks x 256 threads per SM at 64 registers (no spills with
// the quad path's 8 float4 loads in flight; at 48 registers it spills).
template <bool kAdam>
__global__ void __launch_bounds__(256, 4) segments_kernel(const __grid_constant__ SegmentTable t) {
  __shared__ float4 acc_s[8][32];
  __shared__ float red_s[256];
  __shared__ float sum_s[kSegElems];  // the block's summed elements (fused Adam)
  pdl_trigger();
  pdl_wait();
  int si = 0;
  while (si + 1 < t.nseg && (int)blockIdx.x >= t.first_block[si + 1]) ++si;
  const Segment& sg = t.s[si];
  if (seg_quad(sg)) {
    const int i0 = (blockIdx.x - t.first_block[si]) * kQuadElems + threadIdx.x * 4;
    if (i0 >= sg.len) return;
    const float* src = sg.src + i0;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int p0 = 0; p0 < kQuadParts; p0 += 8) {  // 8 parts in flight per round trip
      if (p0 >= sg.nparts) break;
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (p0 + u < sg.nparts) v[u] = __ldcs(reinterpret_cast<const float4*>(src + (long long)(p0 + u) * sg.stride));
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (p0 + u < sg.nparts) {
          acc.x += v[u].x;
          acc.y += v[u].y;
          acc.z += v[u].z;
          acc.w += v[u].w;
        }
    }
    *reinterpret_cast<float4*>(sg.dst + i0) = acc;
    if (kAdam && sg.param_off >= 0) {
      const SegAdam& a = t.adam;
      const long long st = a.ctl->adam_step0 + a.step_in_iter;
      const float bc1 = a.bc[2 * st], bc2 = a.bc[2 * st + 1];
      const long long i = sg.param_off + i0;
      adam_elem(a, i, acc.x, bc1, bc2);
      adam_elem(a, i + 1, acc.y, bc1, bc2);
      adam_elem(a, i + 2, acc.z, bc1, bc2);
      adam_elem(a, i + 3, acc.w, bc1, bc2);
    }
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int base = (blockIdx.x - t.first_block[si]) * kSegElems;
  const bool vec = ((sg.len | (int)(sg.stride & 3)) & 3) == 0 &&
                   ((reinterpret_cast<uintptr_t>(sg.src) | reinterpret_cast<uintptr_t>(sg.dst)) & 15) == 0;
  if (vec) {
    const int i0 = base + lane * 4;
    const int p0 = warp * sg.nparts / 8, p1 = (warp + 1) * sg.nparts / 8;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i0 < sg.len) {
      const float* src = sg.src + i0;
      for (int p = p0; p < p1; p += 4) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (p + u < p1) v[u] = __ldcs(reinterpret_cast<const float4*>(src + (long long)(p + u) * sg.stride));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (p + u < p1) {
            acc.x += v[u].x;
            acc.y += v[u].y;
            acc.z += v[u].z;
            acc.w += v[u].w;
          }
        }
      }
    }
    acc_s[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && i0 < sg.len) {
      float4 s = acc_s[0][lane];
#pragma unroll
      for (int w = 1; w < 8; ++w) {
        const float4 v = acc_s[w][lane];
        s.x += v.x;
        s.y += v.y;
        s.z += v.z;
        s.w += v.w;
      }
      *reinterpret_cast<float4*>(sg.dst + i0) = s;
      *reinterpret_cast<float4*>(sum_s + lane * 4) = s;
    }
  } else {
    const int E = min(kSegElems, sg.len - base);
    int ep = 1;
    while (ep < E) ep <<= 1;
    const int G = 256 / ep;
    const int e = threadIdx.x & (ep - 1), g = threadIdx.x / ep;
    float acc = 0.f;
    if (e < E) {
      const float* src = sg.src + base + e;
      for (int p = g; p < sg.nparts; p += 4 * G) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (p + u * G < sg.nparts) v[u] = __ldcs(src + (long long)(p + u * G) * sg.stride);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (p + u * G < sg.nparts) acc += v[u];
      }
    }
    red_s[threadIdx.x] = acc;
    __syncthreads();
    if (int(threadIdx.x) < E) {
      float s = red_s[threadIdx.x];
      for (int gg = 1; gg < G; ++gg) s += red_s[gg * ep + threadIdx.x];
      sg.dst[base + threadIdx.x] = s;
      sum_s[threadIdx.x] = s;
    }
  }
  if (kAdam && sg.param_off >= 0) {  // fused Adam, same arithmetic as adam_kernel
    __syncthreads();
    const int e = threadIdx.x;  // element of this block
    const int ie = base + e;
    if (e < kSegElems && ie < sg.len) {
      const SegAdam& a = t.adam;
      const long long st = a.ctl->adam_step0 + a.step_in_iter;
      adam_elem(a, sg.param_off + ie, sum_s[e], a.bc[2 * st], a.bc[2 * st + 1]);
    }
  }
}

}  // namespace

int head_loss_blocks(int B) { return (B + 255) / 256; }

void launch_head_loss(const HeadLossArgs& a, cudaStream_t s) {
  if (a.A > kMaxAct) invalid("act_dim > 31 unsupported by the loss kernel");
  const int blocks = head_loss_blocks(a.B);
  if (a.A <= 8)
    launch_pdl(head_loss_kernel<8>, dim3(blocks), dim3(256), 0, s, a);
  else if (a.A <= 16)
    launch_pdl(head_loss_kernel<16>, dim3(blocks), dim3(256), 0, s, a);
  else if (a.A <= 24)
    launch_pdl(head_loss_kernel<24>, dim3(blocks), dim3(256), 0, s, a);
  else
    launch_pdl(head_loss_kernel<31>, dim3(blocks), dim3(256), 0, s, a);
}

int colsum_blocks(int rows) { return (rows + kColsumRows - 1) / kColsumRows; }

void launch_colsum(const __nv_bfloat16* const* D, const int* widths, float* const* partial, int np, int rows,
                   cudaStream_t s) {
  if (np > 16) invalid("too many column-sum problems");
  ColsumArgs a{};
  for (int i = 0; i < np; ++i) {
    if (widths[i] % 32 || widths[i] > 1024) invalid("column-sum width must be a multiple of 32, <= 1024");
    a.D[i] = D[i];
    a.out[i] = partial[i];
    a.width[i] = widths[i];
  }
  launch_pdl(colsum_kernel, dim3(colsum_blocks(rows), np), dim3(256), 0, s, a, rows);
}

void launch_segments(const Segment* segs, int n, cudaStream_t s, const SegAdam* adam) {
  for (int base = 0; base < n; base += kMaxSegments) {
    SegmentTable t{};
    const int m = std::min(kMaxSegments, n - base);
    t.nseg = m;
    t.has_adam = adam != nullptr;
    if (adam) t.adam = *adam;
    t.first_block[0] = 0;
    for (int i = 0; i < m; ++i) {
      t.s[i] = segs[base + i];
      const int per = seg_quad(t.s[i]) ? kQuadElems : kSegElems;
      t.first_block[i + 1] = t.first_block[i] + (std::max(1, t.s[i].len) + per - 1) / per;
    }
    if (t.has_adam)
      launch_pdl(segments_kernel<true>, dim3(t.first_block[m]), dim3(256), 0, s, t);
    else
      launch_pdl(segments_kernel<false>, dim3(t.first_block[m]), dim3(256), 0, s, t);
  }
}

}  // namespace gmi::ppo
