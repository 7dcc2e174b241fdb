// tcgen05 GEMM for the actor-critic MLP layers (sm_100a).
//
//   D[m][n] = sum_k A(m,k) * B(n,k)        bf16 operands, fp32 accumulation in TMEM
//
// Operands arrive by TMA (128B swizzle) into a STAGES-deep shared-memory ring; one
// elected thread issues tcgen05.mma (M = 128, N = BLOCK_N, K = 16 per instruction);
// the four warps then drain TMEM through a fused epilogue. Either operand may be
// K-major (row-major [rows x K]) or MN-major (row-major [K x rows]); the MN-major form
// lets the weight-gradient GEMM (dW = dPre^T * H, reduction over the minibatch rows)
// read the forward activations in place without a transpose pass.
//
// Epilogues (one per MLP use):
//   EPI_BIAS_ELU  hidden-layer forward: bf16 out = elu(acc + bias[n])
//   EPI_DACT      hidden-layer backward: bf16 out = acc * elu'(H[m][n]) with H the
//                 post-activation of the same unit (elu' = 1 if H > 0 else H + 1)
//   EPI_F32       fp32 out (split-K slabs for the weight gradient, reduced later)
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

#include "gemm_types.hpp"
#include "ptx.cuh"

namespace gmi {

__device__ __forceinline__ float elu_f(float x) { return x > 0.f ? x : expm1f(x); }

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int BLOCK_N, int STAGES, int A_MN, int B_MN, int EPI>
__global__ void __launch_bounds__(128, 1) gemm_tcgen05_kernel(const __grid_constant__ GemmParams P) {
  static_assert(BLOCK_N % 64 == 0 && BLOCK_N <= 256, "BLOCK_N must be a multiple of 64, <= 256");
  constexpr uint32_t kABytes = kGemmBlockM * kGemmBlockK * 2;  // 16 KB
  constexpr uint32_t kBBytes = BLOCK_N * kGemmBlockK * 2;
  constexpr uint32_t kStageBytes = kABytes + kBBytes;
  constexpr uint32_t kTmemCols = BLOCK_N < 32 ? 32 : BLOCK_N;
  constexpr uint32_t kIdesc = ptx::umma_idesc_bf16(kGemmBlockM, BLOCK_N, A_MN, B_MN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* acc_bar = empty_bar + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_bar + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int z = blockIdx.z;
  const int prob_idx = z / P.splits;
  const int split = z % P.splits;
  const GemmProblem& pr = P.prob[prob_idx];
  const int m0 = blockIdx.x * kGemmBlockM;
  const int n0 = blockIdx.y * BLOCK_N;
  if (m0 >= pr.M || n0 >= pr.N) return;  // uniform per CTA

  const int nkb_total = (pr.K + kGemmBlockK - 1) / kGemmBlockK;
  const int kb_begin = split * pr.kb_per_split;
  int kb_end = kb_begin + pr.kb_per_split;
  if (kb_end > nkb_total) kb_end = nkb_total;
  const int nkb = kb_end > kb_begin ? kb_end - kb_begin : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    ptx::mbar_init(acc_bar, 1);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&pr.map_a);
    ptx::tma_prefetch_desc(&pr.map_b);
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (nkb > 0) {
    if (warp == 0 && lane == 0) {
      // ---------------- TMA producer
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        if (i >= STAGES) ptx::mbar_wait(&empty_bar[s], ((i / STAGES) - 1) & 1);
        uint8_t* sa = smem + s * kStageBytes;
        uint8_t* sb = sa + kABytes;
        const int k0 = (kb_begin + i) * kGemmBlockK;
        ptx::mbar_arrive_expect_tx(&full_bar[s], kStageBytes);
        if constexpr (A_MN) {
#pragma unroll
          for (int j = 0; j < kGemmBlockM / 64; ++j)
            ptx::tma_load_2d(sa + j * 8192, &pr.map_a, &full_bar[s], m0 + 64 * j, k0 + pr.a_row0);
        } else {
          ptx::tma_load_2d(sa, &pr.map_a, &full_bar[s], k0, m0 + pr.a_row0);
        }
        if constexpr (B_MN) {
#pragma unroll
          for (int j = 0; j < BLOCK_N / 64; ++j)
            ptx::tma_load_2d(sb + j * 8192, &pr.map_b, &full_bar[s], n0 + 64 * j, k0 + pr.b_row0);
        } else {
          ptx::tma_load_2d(sb, &pr.map_b, &full_bar[s], k0, n0 + pr.b_row0);
        }
      }
    } else if (warp == 1 && lane == 0) {
      // ---------------- MMA issuer
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        ptx::mbar_wait(&full_bar[s], (i / STAGES) & 1);
        ptx::tc_fence_after();
        const uint32_t sa = ptx::smem_u32(smem + s * kStageBytes);
        const uint32_t sb = sa + kABytes;
#pragma unroll
        for (int k = 0; k < kGemmBlockK / 16; ++k) {
          // K-major: step 16 elements (32 B) inside the swizzle atom.
          // MN-major: step 16 rows = two 8-row core groups (2 x 1024 B).
          const uint64_t ad = A_MN ? ptx::umma_desc_sw128(sa + k * 2048, 8192, 1024)
                                   : ptx::umma_desc_sw128(sa + k * 32, 16, 1024);
          const uint64_t bd = B_MN ? ptx::umma_desc_sw128(sb + k * 2048, 8192, 1024)
                                   : ptx::umma_desc_sw128(sb + k * 32, 16, 1024);
          ptx::mma_bf16(tmem_base, ad, bd, kIdesc, (i > 0 || k > 0) ? 1u : 0u);
        }
        ptx::mma_commit(&empty_bar[s]);
      }
      ptx::mma_commit(acc_bar);
    }
    __syncwarp();
    ptx::mbar_wait(acc_bar, 0);
    ptx::tc_fence_after();
  }
  __syncwarp();

  // ---------------- epilogue: warp w owns TMEM lanes / tile rows [32w, 32w + 32)
  const int row = m0 + warp * 32 + lane;
  const bool row_ok = row < pr.M;
#pragma unroll 1
  for (int c = 0; c < BLOCK_N / 32; ++c) {
    const int col0 = n0 + c * 32;
    uint32_t r[32];
    if (nkb > 0) {
      ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + c * 32, r);
      ptx::tmem_ld_wait();
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) r[j] = 0u;
    }
    if (!row_ok || col0 >= pr.N) continue;
    if constexpr (EPI == EPI_F32) {
      float* o = reinterpret_cast<float*>(pr.out) + split * pr.split_stride + row * pr.ld_out + col0;
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(o + j) =
            make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                        __uint_as_float(r[j + 3]));
    } else {
      uint32_t packed[16];
      if constexpr (EPI == EPI_BIAS_ELU) {
        const float* b = pr.bias + col0;
#pragma unroll
        for (int j = 0; j < 32; j += 2)
          packed[j / 2] = pack_bf16(elu_f(__uint_as_float(r[j]) + b[j]),
                                    elu_f(__uint_as_float(r[j + 1]) + b[j + 1]));
      } else {  // EPI_DACT
        const uint4* hp = reinterpret_cast<const uint4*>(pr.aux + row * pr.ld_aux + col0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 hv = hp[q];
          const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            __nv_bfloat162 h2 = *reinterpret_cast<const __nv_bfloat162*>(&hw[e]);
            const float h0 = __bfloat162float(h2.x), h1 = __bfloat162float(h2.y);
            const int j = q * 8 + e * 2;
            const float g0 = __uint_as_float(r[j]) * (h0 > 0.f ? 1.f : h0 + 1.f);
            const float g1 = __uint_as_float(r[j + 1]) * (h1 > 0.f ? 1.f : h1 + 1.f);
            packed[j / 2] = pack_bf16(g0, g1);
          }
        }
      }
      uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(pr.out) + row * pr.ld_out + col0);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        o[q] = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc(tmem_base, kTmemCols);
}

template <int BLOCK_N, int STAGES>
constexpr int gemm_smem_bytes() {
  return STAGES * (kGemmBlockM * kGemmBlockK * 2 + BLOCK_N * kGemmBlockK * 2) + 1024 + 256;
}

}  // namespace gmi
