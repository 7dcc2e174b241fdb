// Fused value pass: V = value_net(obs) for every (T+1) x N rollout observation in one
// persistent launch. Each CTA walks 128-row tiles of X_roll and runs the whole value MLP on
// chip -- observation tile (TMA) -> tcgen05.mma with weights streamed through a 3-stage TMA
// ring -> double-buffered TMEM -> 16 epilogue warps bias + ELU back into the next layer's
// SW128 operand tile (half-tile barriers let layer l+1's MMA start while layer l drains) ->
// value head (N = 16, column 0) -> V. Hidden activations never reach HBM (the per-layer
// path wrote and re-read ~4 x 70 MB of them per iteration). Same arithmetic as the per-layer
// GEMM path (same operands, MMA K order and bias_elu2), so V is bit-identical to it.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../host/errors.hpp"
#include "gemm.cuh"
#include "launch.cuh"
#include "rollout.cuh"

namespace gmi::ppo {

namespace {

constexpr int kRows = 128;
constexpr int kEpiWarps = 16;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kStages = 3;
constexpr uint32_t kChunk = kRows * 128;
constexpr uint32_t kActBytes = 4 * kChunk;
constexpr uint32_t kWStage = 256 * 128;
constexpr uint32_t kSmem = 2 * kActBytes + kStages * kWStage + 256 + 1024;

// WIDE: hidden widths up to 512 with the shared-memory / TMEM plan a.plan (rollout.cuh), as
// rollout_kernel<.., true>: 128-row weight parts, act_rdy[pair] per K-chunk pair, and hd_free
// (the head accumulator read) before the next tile's layer 0 when their TMEM columns overlap.
template <bool WIDE>
__global__ void __launch_bounds__(kThreads, 1) value_mlp_kernel(const __grid_constant__ ValueArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::align_smem_1024(smem_raw);
  const WidePlan& P = a.plan;
  uint8_t* act_buf0 = smem;
  uint8_t* act_buf1 = smem + kActBytes;
  uint8_t* wring = WIDE ? smem + P.ring_off : smem + 2 * kActBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(WIDE ? smem + P.bar_off : wring + kStages * kWStage);
  uint64_t* wfull = bars;
  uint64_t* wempty = bars + (WIDE ? 8 : kStages);
  uint64_t* obs_full = bars + (WIDE ? 16 : 2 * kStages);
  uint64_t* obs_free = obs_full + 1;
  uint64_t* acc_full = obs_free + 1;
  uint64_t* act_lo = acc_full + 1;
  uint64_t* act_hi = act_lo + 1;
  uint64_t* act_rdy = act_lo;       // WIDE: [4]
  uint64_t* hd_free = act_lo + 4;   // WIDE: head accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(act_lo + 5);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = a.L;
  const int ntiles = (a.rows + kRows - 1) / kRows;
  // the last MMA of a tile that reads the observation tile (act_buf0 = even layers; WIDE: layer 0
  // from its own buffer, else the head, the last reader of the in-place region)
  const int last_even = WIDE ? (P.obs_sep ? 0 : L) : (L % 2 == 0) ? L : L - 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < (WIDE ? P.nstages : kStages); ++s) {
      ptx::mbar_init(&wfull[s], 1);
      ptx::mbar_init(&wempty[s], 1);
    }
    ptx::mbar_init(obs_full, 1);
    ptx::mbar_init(obs_free, 1);
    ptx::mbar_init(acc_full, 1);
    for (int p = 0; p < (WIDE ? 4 : 2); ++p) ptx::mbar_init(&act_rdy[p], kEpiWarps);
    ptx::mbar_init(hd_free, kEpiWarps);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&a.map_obs);
    for (int l = 0; l <= L; ++l) ptx::tma_prefetch_desc(&a.map_w[l]);
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  pdl_trigger();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      const int nobs = (a.in_p[0] + 63) / 64;
      int it = 0, ti = 0;
      for (int j = blockIdx.x; j < ntiles; j += gridDim.x, ++ti) {
        if (ti > 0) ptx::mbar_wait_sleep(obs_free, (ti - 1) & 1);
        ptx::mbar_arrive_expect_tx(obs_full, nobs * kChunk);
        for (int kc = 0; kc < nobs; ++kc)
          ptx::tma_load_2d(smem + (WIDE ? P.in_off[0] : 0u) + kc * kChunk, &a.map_obs, obs_full, kc * 64, j * kRows);
        for (int l = 0; l <= L && WIDE; ++l) {  // one [<=128 rows x 64 K] box per (K-chunk, N part)
          const int nk = (a.in_p[l] + 63) / 64, np = (a.out_n[l] + 127) / 128;
          const uint32_t bytes = uint32_t(P.wrows[l]) * 128u;
          for (int kc = 0; kc < nk; ++kc)
            for (int p = 0; p < np; ++p, ++it) {
              const int s = it % P.nstages;
              if (it >= P.nstages) ptx::mbar_wait_sleep(&wempty[s], ((it / P.nstages) - 1) & 1);
              ptx::mbar_arrive_expect_tx(&wfull[s], bytes);
              ptx::tma_load_2d(wring + s * kWideStage, &a.map_w[l], &wfull[s], kc * 64, p * 128);
            }
        }
        for (int l = 0; l <= L && !WIDE; ++l) {
          const int nk = (a.in_p[l] + 63) / 64;
          const uint32_t bytes = uint32_t(a.out_n[l]) * 128u;
          for (int kc = 0; kc < nk; ++kc, ++it) {
            const int s = it % kStages;
            if (it >= kStages) ptx::mbar_wait_sleep(&wempty[s], ((it / kStages) - 1) & 1);
            ptx::mbar_arrive_expect_tx(&wfull[s], bytes);
            ptx::tma_load_2d(wring + s * kWStage, &a.map_w[l], &wfull[s], kc * 64, 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0 && WIDE) {
      int it = 0, ti = 0;
      uint32_t ph[4] = {0u, 0u, 0u, 0u};
      for (int j = blockIdx.x; j < ntiles; j += gridDim.x, ++ti)
        for (int l = 0; l <= L; ++l) {
          const int K = a.in_p[l], nk = (K + 63) / 64, N = a.out_n[l], np = (N + 127) / 128;
          const uint32_t in = ptx::smem_u32(smem + P.in_off[l]);
          const uint32_t acc = tmem + uint32_t(P.tmem[l]);
          int ready = 0;
          if (l == 0) {
            ptx::mbar_wait(obs_full, ti & 1);
            if (ti > 0 && P.wrap) ptx::mbar_wait(hd_free, (ti - 1) & 1);
          } else if (P.drain[l]) {
            for (; ready < (nk + 1) / 2; ++ready) ptx::mbar_wait(&act_rdy[ready], (ph[ready]++) & 1);
          }
          for (int kc = 0; kc < nk; ++kc) {
            if (l > 0 && (kc >> 1) == ready) {
              ptx::mbar_wait(&act_rdy[ready], (ph[ready]++) & 1);
              ++ready;
            }
            const int ks = min(4, (K - kc * 64 + 15) / 16);
            for (int p = 0; p < np; ++p, ++it) {
              const int s = it % P.nstages;
              ptx::mbar_wait(&wfull[s], (it / P.nstages) & 1);
              ptx::tc_fence_after();
              const uint32_t wb = ptx::smem_u32(wring + s * kWideStage);
              const uint32_t idesc = ptx::umma_idesc_bf16(kRows, uint32_t(min(128, N - p * 128)), 0, 0);
              for (int k = 0; k < ks; ++k)
                ptx::mma_bf16(acc + p * 128, ptx::umma_desc_sw128(in + kc * kChunk + k * 32, 16, 1024),
                              ptx::umma_desc_sw128(wb + k * 32, 16, 1024), idesc, (kc > 0 || k > 0) ? 1u : 0u);
              ptx::mma_commit(&wempty[s]);
            }
          }
          ptx::mma_commit(acc_full);
          if (l == last_even) ptx::mma_commit(obs_free);  // the observation tile may be reloaded
        }
    }
    if (lane == 0 && !WIDE) {
      int it = 0, ph_lo = 0, ph_hi = 0, acc_ph = 0, ti = 0;
      for (int j = blockIdx.x; j < ntiles; j += gridDim.x, ++ti)
        for (int l = 0; l <= L; ++l, ++acc_ph) {
          const uint32_t acc = tmem + (acc_ph & 1) * 256;
          const uint32_t idesc = ptx::umma_idesc_bf16(kRows, uint32_t(a.out_n[l]), 0, 0);
          const uint32_t in = ptx::smem_u32((l & 1) ? act_buf1 : act_buf0);
          const int K = a.in_p[l];
          const int nk = (K + 63) / 64;
          if (l == 0) ptx::mbar_wait(obs_full, ti & 1);
          for (int kc = 0; kc < nk; ++kc, ++it) {
            if (l > 0 && kc == 0) ptx::mbar_wait(act_lo, (ph_lo++) & 1);
            if (l > 0 && kc == 2) ptx::mbar_wait(act_hi, (ph_hi++) & 1);
            const int s = it % kStages;
            ptx::mbar_wait(&wfull[s], (it / kStages) & 1);
            ptx::tc_fence_after();
            const uint32_t wb = ptx::smem_u32(wring + s * kWStage);
            const int ks = min(4, (K - kc * 64 + 15) / 16);
            for (int k = 0; k < ks; ++k)
              ptx::mma_bf16(acc, ptx::umma_desc_sw128(in + kc * kChunk + k * 32, 16, 1024),
                            ptx::umma_desc_sw128(wb + k * 32, 16, 1024), idesc, (kc > 0 || k > 0) ? 1u : 0u);
            ptx::mma_commit(&wempty[s]);
          }
          if (l > 0 && nk <= 2) ptx::mbar_wait(act_hi, (ph_hi++) & 1);  // keep the phases paired
          ptx::mma_commit(acc_full);
          if (l == last_even) ptx::mma_commit(obs_free);  // the observation tile may be reloaded
        }
    }
  } else {
    // ------------------------------------------------ epilogue warps
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    int accph = 0;
    for (int j = blockIdx.x; j < ntiles; j += gridDim.x) {
      for (int l = 0; l < L; ++l) {
        const uint32_t acc = WIDE ? tmem + uint32_t(P.tmem[l]) : tmem + (accph & 1) * 256;
        ptx::mbar_wait_sleep(acc_full, accph & 1);
        ++accph;
        ptx::tc_fence_after();
        uint8_t* out = WIDE ? smem + P.in_off[l + 1] : (l & 1) ? act_buf0 : act_buf1;
        const float* bias = a.bias[l];
        const int nchunks = a.out_n[l] / 32;
        const int npass = WIDE ? (a.out_n[l] + 127) / 128 : 2;
#pragma unroll 1
        for (int pass = 0; pass < npass; ++pass) {
          const int c = h + 4 * pass;
          if (c < nchunks) {
            uint32_t r[32];
            ptx::tmem_ld_32x32b_x32(acc + (static_cast<uint32_t>(q * 32) << 16) + c * 32, r);
            const float4* b4 = reinterpret_cast<const float4*>(bias + c * 32);
            ptx::tmem_ld_wait();
            uint32_t packed[16];
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const float4 b = __ldg(b4 + jj);
              const float2 y0 = bias_elu2(make_float2(__uint_as_float(r[4 * jj]), __uint_as_float(r[4 * jj + 1])),
                                          make_float2(b.x, b.y));
              const float2 y1 = bias_elu2(
                  make_float2(__uint_as_float(r[4 * jj + 2]), __uint_as_float(r[4 * jj + 3])), make_float2(b.z, b.w));
              packed[2 * jj] = pack_bf16(y0.x, y0.y);
              packed[2 * jj + 1] = pack_bf16(y1.x, y1.y);
            }
            uint8_t* chunk = out + (c >> 1) * kChunk + row * 128;
            const int u0 = (c & 1) * 4;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              *reinterpret_cast<uint4*>(chunk + (((u0 + u) ^ (row & 7)) << 4)) =
                  make_uint4(packed[4 * u], packed[4 * u + 1], packed[4 * u + 2], packed[4 * u + 3]);
          }
          ptx::fence_proxy_async_smem();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(WIDE ? &act_rdy[pass] : pass == 0 ? act_lo : act_hi);
        }
      }
      // ---- value head: V = acc[:, 0] + b_v
      const uint32_t hacc = WIDE ? tmem + uint32_t(P.tmem[L]) : tmem + (accph & 1) * 256;
      ptx::mbar_wait_sleep(acc_full, accph & 1);
      ++accph;
      ptx::tc_fence_after();
      if (h == 0) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(hacc + (static_cast<uint32_t>(q * 32) << 16), r);
        ptx::tmem_ld_wait();
        const long long grow = (long long)j * kRows + row;
        if (grow < a.rows) a.V[grow] = __uint_as_float(r[0]) + a.bias[L][0];
      }
      ptx::tc_fence_before();
      if constexpr (WIDE) {
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(hd_free);
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

}  // namespace

bool value_wide_fusable(int L, const int* widths_p, WidePlan* plan) {
  return plan_wide(L, widths_p, 16, false, plan);
}

void launch_value_mlp(const ValueArgs& a, int max_ctas, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    GMI_CUDA_CHECK(cudaFuncSetAttribute(value_mlp_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    GMI_CUDA_CHECK(cudaFuncSetAttribute(value_mlp_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    configured = true;
  }
  const int tiles = (a.rows + kRows - 1) / kRows;
  const dim3 grid(std::max(1, std::min(tiles, max_ctas)));
  if (a.wide)
    launch_pdl(value_mlp_kernel<true>, grid, dim3(kThreads), a.plan.smem, s, a);
  else
    launch_pdl(value_mlp_kernel<false>, grid, dim3(kThreads), kSmem, s, a);
}

}  // namespace gmi::ppo
