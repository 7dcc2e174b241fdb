// Fused training forward of one PPO minibatch (K4 + K6 + the head parts of K7):
// for each 128-row tile of the epoch copy X_sh, on one net (CTA b serves net b % 2),
//   hidden layers   H_l = elu(H_{l-1} W_l^T + b_l) on chip: observation tile (TMA) ->
//                   tcgen05.mma with the layer weights streamed through a 3-stage TMA ring ->
//                   double-buffered TMEM -> 16 epilogue warps bias + ELU back into the next
//                   layer's SW128 operand tile; H_1..H_{L-1} are also TMA-stored for the
//                   backward GEMMs straight from those operand tiles (H_L never leaves the SM)
//   head MMA1       mu | v = H_L W_head^T                       (N = 16 / 32)
//   loss            clipped surrogate / value loss per row -> G (bf16 operand tile)
//   MMA2            G W_head                                   (N = hp)
//   MMA3            H_L^T G, the tile's head weight gradient   (drained into registers)
//   dact epilogue   dPre_L = (G W_head) * elu'(H_L), written in place over H_L and TMA-stored
// so the per-layer forward GEMMs and the fused head kernel (head_fused.cu) become one launch,
// and the H_L round trip through HBM disappears. Per-CTA outputs (head weight-gradient slab,
// db_head / dlog_std / loss-statistic records) have exactly the fused head kernel's layout,
// so the gradient assembly is unchanged. Numerics follow value_mlp.cu (forward) and
// head_fused.cu (loss, dact); the head weight gradient is summed per tile in fp32 registers.
//
// Shared memory: act_buf0 / act_buf1 (64 KB each, [4 K-chunks][128 rows][128 B] SW128) +
// 3 x 32 KB weight ring = 224 KB. G lives in K-chunk 3 of act_buf0 (free between the last
// MMA that reads H_{L-1} and the next tile's layer-1 epilogue); the next observation tile
// is prefetched into chunk(s) 0..2 of act_buf0 meanwhile. Hence L odd (1 or 3), S_p <= 192.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../host/errors.hpp"
#include "gemm.cuh"
#include "launch.cuh"
#include "ppo_common.cuh"
#include "head_loss.cuh"
#include "train_fwd.cuh"

namespace gmi::ppo {

namespace {

constexpr int kRows = 128;
constexpr int kEpiWarps = 16;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kStages = 3;
constexpr uint32_t kChunk = kRows * 128;  // [128 rows][64 bf16], SW128
constexpr uint32_t kActBytes = 4 * kChunk;
constexpr uint32_t kWStage = 256 * 128;
constexpr uint32_t kOffBar = 2 * kActBytes + kStages * kWStage;
constexpr int kQ = 68;                                 // per-quarter loss record: sums [0, 64) + statistics
constexpr uint32_t kOffLacc = kOffBar + 640;  // after barriers (128 B) + 128 per-action constants
constexpr uint32_t kSmem = kOffLacc + 4 * kQ * 4 + 1024;  // barriers + constants + records + alignment
static_assert(kSmem <= 232448, "shared memory budget");

// Development trace (tools/train_fwd_trace.py): compiled in only with `make TRACE=1`.
__device__ __forceinline__ void stamp(unsigned long long* tr, int ti, int k) {
#ifdef GMI_TRACE
  if (tr && blockIdx.x == 0 && ti < 4) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[ti * 16 + k] = t;
  }
#else
  (void)tr, (void)ti, (void)k;
#endif
}

__device__ __forceinline__ void pair_bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory"); }

template <int MAXA>
__global__ void __launch_bounds__(kThreads, 1) train_fwd_kernel(const __grid_constant__ TrainFwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::align_smem_1024(smem_raw);
  uint8_t* buf0 = smem;
  uint8_t* buf1 = smem + kActBytes;
  uint8_t* wring = smem + 2 * kActBytes;
  uint8_t* sG = buf0 + 3 * kChunk;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* wfull = bars;
  uint64_t* wempty = bars + kStages;
  uint64_t* obs_full = bars + 2 * kStages;
  uint64_t* obs_free = obs_full + 1;
  uint64_t* acc_full = obs_full + 2;
  uint64_t* act_lo = obs_full + 3;
  uint64_t* act_hi = obs_full + 4;
  uint64_t* g_ready = obs_full + 5;
  uint64_t* dw_drained = obs_full + 6;
  uint64_t* h_stored = obs_full + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(obs_full + 8);
  float* cst = reinterpret_cast<float*>(smem + kOffBar + 128);  // log_std, exp(log_std), head bias
  float* red = reinterpret_cast<float*>(smem + kOffLacc);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int net = blockIdx.x & 1;
  const int cta = blockIdx.x >> 1, ctas = gridDim.x >> 1;
  const TrainFwdNet& nw = a.net[net];
  const int L = a.L, hp = a.hp, NH = nw.nh, nout = nw.n_out;
  const int mtiles = (a.Bm + kRows - 1) / kRows;
  const int nobs = (a.S_p + 63) / 64;
  const int nkh = (hp + 63) / 64;
  const int last_even = L - 1;  // L odd: the last MMA reading act_buf0 (H_{L-1}, or X when L = 1)
  const bool stores_buf0 = L >= 3;  // H_2 is stored from act_buf0

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&wfull[s], 1);
      ptx::mbar_init(&wempty[s], 1);
    }
    ptx::mbar_init(obs_full, 1);
    ptx::mbar_init(obs_free, 1);
    ptx::mbar_init(acc_full, 1);
    ptx::mbar_init(act_lo, kEpiWarps);
    ptx::mbar_init(act_hi, kEpiWarps);
    ptx::mbar_init(g_ready, 4);
    ptx::mbar_init(dw_drained, kEpiWarps);
    ptx::mbar_init(h_stored, kEpiWarps / 2);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&a.map_x);
    for (int l = 0; l <= L; ++l) ptx::tma_prefetch_desc(&nw.map_w[l]);
    ptx::tma_prefetch_desc(&nw.map_wm);
    ptx::tma_prefetch_desc(&nw.map_d);
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
      int it = 0, ti = 0;
      auto stage = [&](uint32_t bytes) {
        const int s = it % kStages;
        if (it >= kStages) ptx::mbar_wait_sleep(&wempty[s], ((it / kStages) - 1) & 1);
        ptx::mbar_arrive_expect_tx(&wfull[s], bytes);
        ++it;
        return s;
      };
      for (int j = cta; j < mtiles; j += ctas, ++ti) {
        if (ti > 0) {
          ptx::mbar_wait_sleep(obs_free, (ti - 1) & 1);
          if (stores_buf0) ptx::mbar_wait_sleep(h_stored, (ti - 1) & 1);  // H_2 store has read act_buf0
        }
        ptx::mbar_arrive_expect_tx(obs_full, uint32_t(nobs) * kChunk);
        for (int kc = 0; kc < nobs; ++kc)
          ptx::tma_load_2d(buf0 + kc * kChunk, &a.map_x, obs_full, kc * 64, int(a.row0) + j * kRows);
        for (int l = 0; l <= L; ++l) {
          const int nk = (nw.in_p[l] + 63) / 64;
          for (int kc = 0; kc < nk; ++kc) {
            const int s = stage(uint32_t(nw.out_n[l]) * 128u);
            ptx::tma_load_2d(wring + s * kWStage, &nw.map_w[l], &wfull[s], kc * 64, 0);
          }
        }
        // head weights viewed [K = NH rows][N = hp] (MN-major B of MMA2), nkh boxes of [32][64]
        const int s = stage(uint32_t(nkh) * 4096u);
        for (int kc = 0; kc < nkh; ++kc)
          ptx::tma_load_2d(wring + s * kWStage + kc * 4096, &nw.map_wm, &wfull[s], kc * 64, 0);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc2 = ptx::umma_idesc_bf16(kRows, uint32_t((hp + 15) / 16 * 16), 0, 1);
      const uint32_t idesc3 = ptx::umma_idesc_bf16(kRows, uint32_t(NH), 1, 1);
      const uint32_t g0 = ptx::smem_u32(sG);
      const uint32_t hl = ptx::smem_u32((L & 1) ? buf1 : buf0);
      int it = 0, ph_lo = 0, ph_hi = 0, u = 0, ti = 0;
      for (int j = cta; j < mtiles; j += ctas, ++ti) {
        if (ti > 0) ptx::mbar_wait(dw_drained, (ti - 1) & 1);  // the head / MMA3 buffer is free again
        for (int l = 0; l <= L; ++l, ++u) {
          const uint32_t acc = tmem + (u & 1) * 256;
          const uint32_t idesc = ptx::umma_idesc_bf16(kRows, uint32_t(nw.out_n[l]), 0, 0);
          const uint32_t in = ptx::smem_u32((l & 1) ? buf1 : buf0);
          const int K = nw.in_p[l];
          const int nk = (K + 63) / 64;
          if (l == 0) {
            ptx::mbar_wait(obs_full, ti & 1);
            stamp(a.trace, ti, 11);
          }
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
          if (l == last_even) ptx::mma_commit(obs_free);
        }
        // MMA2 (G W_head -> acc[u]) and MMA3 (H_L^T G -> the head buffer's first 64 columns)
        const uint32_t hb = tmem + ((u - 1) & 1) * 256;
        const uint32_t acc2 = tmem + (u & 1) * 256;
        ptx::mbar_wait(g_ready, ti & 1);
        stamp(a.trace, ti, 12);
        const int s = it % kStages;
        ptx::mbar_wait(&wfull[s], (it / kStages) & 1);
        ptx::tc_fence_after();
        const uint32_t wm0 = ptx::smem_u32(wring + s * kWStage);
        for (int k = 0; k < NH / 16; ++k)
          ptx::mma_bf16(acc2, ptx::umma_desc_sw128(g0 + k * 32, 16, 1024),
                        ptx::umma_desc_sw128(wm0 + k * 2048, 4096, 1024), idesc2, k > 0 ? 1u : 0u);
        for (int half = 0; half * 128 < hp; ++half)
          for (int k = 0; k < kRows / 16; ++k)
            ptx::mma_bf16(hb + half * 32, ptx::umma_desc_sw128(hl + 2 * half * kChunk + k * 2048, kChunk, 1024),
                          ptx::umma_desc_sw128(g0 + k * 2048, 8192, 1024), idesc3, k > 0 ? 1u : 0u);
        ptx::mma_commit(&wempty[s]);
        ++it;
        ptx::mma_commit(acc_full);
        ++u;
      }
    }
  } else {
    // ------------------------------------------------ epilogue warps
    const int e = warp - 2;
    const int q = warp & 3;
    const int h = e >> 2;
    const int row = q * 32 + lane;
    const int pair_id = 2 + q * 2 + (h >> 1);  // named barrier of the two warps sharing a 64-col box
    const bool even = (h & 1) == 0;
    const float invB = 1.0f / float(a.Bm);
    const int et = threadIdx.x - 64;
    float* lacc = red + q * kQ;  // this lane quarter's per-action sums [0, 64) and statistics [64, 68)
    if (et < a.A) {
      const float ls = a.log_std[et];
      cst[et] = ls;
      cst[32 + et] = expf(ls);
      cst[96 + et] = 1.0f / expf(ls);
    }
    if (et < nout) cst[64 + et] = nw.bias[L][et];
    if (h == 0 && lane == 0)
      for (int i = 0; i < kQ; ++i) lacc[i] = 0.f;
    epi_bar();
    float st[4] = {0.f, 0.f, 0.f, 0.f};
    float sg[kLossRegAcc<MAXA> ? MAXA : 1], sl[kLossRegAcc<MAXA> ? MAXA : 1];  // running per-action sums (A <= 8)
#pragma unroll
    for (int i = 0; i < (kLossRegAcc<MAXA> ? MAXA : 1); ++i) sg[i] = sl[i] = 0.f;
    float dwacc[16];  // head weight gradient of hidden unit (h >> 1) * 128 + row, outputs (h & 1) * 16 + i
#pragma unroll
    for (int i = 0; i < 16; ++i) dwacc[i] = 0.f;
    // before overwriting a 64-col box that this pair TMA-stored earlier: the store has read it
    auto reuse_box = [&]() {
      if (even && lane == 0) ptx::bulk_wait_read<0>();
      pair_bar(pair_id);
    };
    auto store_box = [&](const CUtensorMap* map, uint8_t* buf, int kc, int grow0) {
      ptx::fence_proxy_async_smem();
      pair_bar(pair_id);
      if (even && lane == 0) {
        ptx::tma_store_2d(map, buf + kc * kChunk + q * 4096, kc * 64, grow0);
        ptx::bulk_commit();
      }
    };
    int accph = 0;
    unsigned long long* tr = (warp == 2 && lane == 0) ? a.trace : nullptr;
    for (int j = cta, ti = 0; j < mtiles; j += ctas, ++ti) {
      const int grow0 = j * kRows + q * 32;  // minibatch row of this warp quarter's first row
      stamp(tr, ti, 0);
      // ---- hidden layers
      for (int l = 0; l < L; ++l) {
        const uint32_t acc = tmem + (accph & 1) * 256;
        const bool store = l < L - 1;
        uint8_t* out = (l & 1) ? buf0 : buf1;
        if (stores_buf0 && l == 2 && even) {  // H_2 (stored from act_buf0 during layer 1) has left smem
          if (lane == 0) {
            ptx::bulk_wait_read<0>();
            ptx::mbar_arrive(h_stored);
          }
        }
        ptx::mbar_wait_sleep(acc_full, accph & 1);
        ++accph;
        stamp(tr, ti, 1 + l);
        ptx::tc_fence_after();
        const float* bias = nw.bias[l];
        const int nchunks = nw.out_n[l] / 32;
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          const int c = h + 4 * pass;
          reuse_box();
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
            for (int uu = 0; uu < 4; ++uu)
              *reinterpret_cast<uint4*>(chunk + (((u0 + uu) ^ (row & 7)) << 4)) =
                  make_uint4(packed[4 * uu], packed[4 * uu + 1], packed[4 * uu + 2], packed[4 * uu + 3]);
          }
          if (store && (c >> 1) * 64 < nw.out_n[l]) store_box(&nw.map_h[l], out, c >> 1, grow0);
          ptx::fence_proxy_async_smem();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(pass == 0 ? act_lo : act_hi);
        }
        stamp(tr, ti, 4 + l);
      }
      // ---- head MMA1 -> per-row loss -> G (column group 0; the other groups go ahead)
      if (h == 0) {
        const long long rr = a.row0 + j * kRows + row;
        const bool valid = j * kRows + row < a.Bm;
        float act_r[kActRegs<MAXA>];
        float oldlp = 0.f, adv = 0.f, ret = 0.f;
        if (valid) {
          if (net == 0) {
            if constexpr (kLossPre<MAXA>) {
#pragma unroll
              for (int i = 0; i < MAXA; ++i)
                if (i < nout) act_r[i] = a.act[rr * nout + i];
            }
            oldlp = a.oldlp[rr];
            adv = a.adv[rr];
          } else {
            ret = a.ret[rr];
          }
        }
        ptx::mbar_wait_sleep(acc_full, accph & 1);
        stamp(tr, ti, 7);
        ptx::tc_fence_after();
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem + (accph & 1) * 256 + (static_cast<uint32_t>(q * 32) << 16), r);
        ptx::tmem_ld_wait();
        // G row into K-chunk 3 of act_buf0 (SW128). The H_2 stores that read that chunk have
        // completed (h_stored, arrived before layer 2).
        head_row_loss<MAXA>(net, r, cst, nout, NH, valid, a.act + rr * nout, act_r, oldlp, adv, ret, a.clip,
                            a.vf_coef, a.ent_coef, invB, sG + row * 128, row, lacc, st, sg, sl);
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(g_ready);
        stamp(tr, ti, 8);
      } else {
        // the other groups still observe the head phase: an mbarrier parity wait is only
        // meaningful for the barrier's current or just-completed phase
        ptx::mbar_wait_sleep(acc_full, accph & 1);
      }
      ++accph;
      // ---- MMA2 / MMA3 landed: drain the tile's head weight gradient, then dPre_L
      const uint32_t hb = tmem + ((accph - 1) & 1) * 256;
      const uint32_t acc2 = tmem + (accph & 1) * 256;
      ptx::mbar_wait_sleep(acc_full, accph & 1);
      ++accph;
      stamp(tr, ti, 9);
      ptx::tc_fence_after();
      {
        const int half = h >> 1, col = half * 32 + (h & 1) * 16;
        if ((h & 1) * 16 < NH && half * 128 < hp) {
          uint32_t r[16];
          ptx::tmem_ld_32x32b_x16(hb + (static_cast<uint32_t>(q * 32) << 16) + col, r);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) dwacc[i] += __uint_as_float(r[i]);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(dw_drained);
      }
      uint8_t* hlb = (L & 1) ? buf1 : buf0;
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        const int c = h + 4 * pass;
        if (c * 32 < hp) {
          uint32_t r[32];
          ptx::tmem_ld_32x32b_x32(acc2 + (static_cast<uint32_t>(q * 32) << 16) + c * 32, r);
          uint8_t* hrow = hlb + (c >> 1) * kChunk + row * 128;
          uint4 hv[4];
#pragma unroll
          for (int uu = 0; uu < 4; ++uu)
            hv[uu] = *reinterpret_cast<const uint4*>(hrow + ((((c & 1) * 4 + uu) ^ (row & 7)) << 4));
          ptx::tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int uu = 0; uu < 4; ++uu) {
            const uint32_t hw[4] = {hv[uu].x, hv[uu].y, hv[uu].z, hv[uu].w};
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              const int jj = uu * 8 + x * 2;
              const float2 d = dact2(make_float2(__uint_as_float(r[jj]), __uint_as_float(r[jj + 1])), hw[x]);
              packed[jj / 2] = pack_bf16(d.x, d.y);
            }
          }
          // in place: this thread's row x 32 columns of H_L become dPre_L
#pragma unroll
          for (int uu = 0; uu < 4; ++uu)
            *reinterpret_cast<uint4*>(hrow + ((((c & 1) * 4 + uu) ^ (row & 7)) << 4)) =
                make_uint4(packed[4 * uu], packed[4 * uu + 1], packed[4 * uu + 2], packed[4 * uu + 3]);
        }
        if ((c >> 1) * 64 < hp) store_box(&nw.map_d, hlb, c >> 1, grow0);
      }
      stamp(tr, ti, 10);
      ptx::tc_fence_before();
    }

    // ---- per-CTA outputs
    // (a) head weight gradient slab [cta][n_out][hp] (hidden unit k = half * 128 + row)
    {
      const int half = h >> 1, o0 = (h & 1) * 16, k = half * 128 + row;
      if (o0 < NH && k < hp)
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (o0 + i < nout) nw.dw_slab[((long long)cta * nout + o0 + i) * hp + k] = dwacc[i];
    }
    // (b) head-bias / log-std gradients and loss statistics: per-quarter records in `red`
    if (lane == 0) ptx::bulk_wait<0>();
    const int stride = head_partial_stride(a.A);
    if (h == 0) head_loss_flush<MAXA>(nout, lacc, st, sg, sl);
    epi_bar();
    if (h == 0 && q == 0)
      for (int col = lane; col < stride; col += 32) {
        int src = -1;  // offset inside a quarter record, or -1 for the other net's fields
        if (net == 0) {
          if (col < a.A) src = col;
          else if (col > a.A && col <= 2 * a.A) src = 32 + col - a.A - 1;
          else if (col == 2 * a.A + 1) src = 64;
          else if (col == 2 * a.A + 3) src = 66;
          else if (col == 2 * a.A + 4) src = 67;
        } else {
          if (col == a.A) src = 0;
          else if (col == 2 * a.A + 2) src = 65;
        }
        a.part[(long long)blockIdx.x * stride + col] =
            src < 0 ? 0.f : ((red[src] + red[kQ + src]) + red[2 * kQ + src]) + red[3 * kQ + src];
      }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

}  // namespace

bool train_fwd_fusable(int L, const int* widths_p, int S_p, int A) {
  if (!(L == 1 || L == 3) || S_p > 192 || A < 1 || A > 31) return false;
  for (int l = 1; l <= L; ++l)
    if (widths_p[l] > 256) return false;
  return true;
}

void launch_train_fwd(const TrainFwdArgs& a, int grid, cudaStream_t s) {
  auto go = [&](auto kern) {
    GMI_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    launch_pdl(kern, dim3(grid), dim3(kThreads), kSmem, s, a);
  };
  if (a.A <= 8)
    go(train_fwd_kernel<8>);
  else if (a.A <= 16)
    go(train_fwd_kernel<16>);
  else
    go(train_fwd_kernel<31>);
}

}  // namespace gmi::ppo
