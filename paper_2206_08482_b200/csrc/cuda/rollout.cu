// Fused rollout: the whole T-step policy rollout of 128 envs in one persistent CTA
// (K3 env step + K4 actor inference of SURVEY §2.2, fused).
//
// Per env step the CTA runs the policy MLP on its 128 env rows entirely on chip and then
// steps the environments:
//   obs (bf16, SW128 K-major in smem) -> [tcgen05.mma, weights streamed by TMA from L2]
//   -> TMEM accumulator -> epilogue warps: bias + ELU -> bf16 back into smem (the next
//   layer's A operand) -> ... -> policy head (N = 16/32) -> mu -> Gaussian sample, log-prob,
//   clipped action, synthetic Ant-like dynamics, reward, integer episode clock / reset ->
//   next observation written straight into the smem operand tile (and to X_roll in HBM for
//   the value pass / update).
// Activations never leave the SM; episode clocks stay in registers for the whole rollout.
// This replaces T x (L hidden GEMMs + head GEMM + act/env kernel) launches whose runtime was
// launch/latency-bound at M = envs per GMI.
//
// Roles: warp 0 = TMA producer (initial obs tile, weight K-chunks through a 3-stage ring),
// warp 1 = single-thread tcgen05.mma issuer, warps 2..17 = epilogue / env threads (4 threads
// per env in the env phase). MMA and epilogue alternate per layer (dependency chain).
//
// Numerics: identical MLP arithmetic to the per-layer GEMM path (same bf16 operands, same
// MMA K order, same bias_elu2); env step formulas as act_env_kernel / oracle/ppo_oracle.c.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "../host/errors.hpp"
#include "gemm.cuh"
#include "launch.cuh"
#include "ppo.cuh"
#include "ppo_common.cuh"
#include "rng.cuh"
#include "rollout.cuh"

namespace gmi::ppo {

namespace {

constexpr float kDt = 0.05f, kDamp = 1.0f, kCouple = 0.1f, kCtrl = 0.1f, kStateC = 0.1f;
constexpr float kTwoPi = 6.28318530717958648f;
constexpr int kRows = 128;
constexpr int kEpiWarps = 16;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kStages = 3;
constexpr uint32_t kChunk = kRows * 128;        // one 64-column K-chunk of a 128-row tile
constexpr uint32_t kActBytes = 4 * kChunk;       // 128 x 256 bf16
constexpr uint32_t kWStage = 256 * 128;          // <= 256 weight rows x 64 K bf16
constexpr int kMuLd = 33;                        // fp32 row pitch of the mu / action staging
constexpr uint32_t kSmemBytes = 2 * kActBytes + kStages * kWStage + 512 + 1024;  // + barriers, std table

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory"); }

// Development trace: globaltimer stamps of one epilogue thread of CTA 0 (a.trace[t * 16 + k]).
__device__ __forceinline__ void trace_at(const RolloutArgs& a, int idx) {
  if (a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[idx] = t;
  }
}

__device__ __forceinline__ uint32_t sw128(int row, int col_bf16) {  // byte offset inside a K-chunk
  const int u = (col_bf16 & 63) >> 3;
  return uint32_t(row * 128 + ((u ^ (row & 7)) << 4) + (col_bf16 & 7) * 2);
}

// MAXB: 4-dim state blocks per env thread (S <= 16 * MAXB).
// WIDE: hidden widths up to 512 (a.plan, rollout.cuh): per-layer tile offsets and TMEM columns,
// weights in 128-row N parts, input K-chunk pairs released by act_rdy[pair] (up to 4 pairs).
template <int MAXB, bool WIDE>
__global__ void __launch_bounds__(kThreads, 1) rollout_kernel(const __grid_constant__ RolloutArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::align_smem_1024(smem_raw);
  const WidePlan& P = a.plan;
  uint8_t* act_buf0 = smem;
  uint8_t* act_buf1 = smem + kActBytes;
  uint8_t* wring = WIDE ? smem + P.ring_off : smem + 2 * kActBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(WIDE ? smem + P.bar_off : wring + kStages * kWStage);
  uint64_t* wfull = bars;
  uint64_t* wempty = bars + (WIDE ? 8 : kStages);
  uint64_t* obs_bar = bars + (WIDE ? 16 : 2 * kStages);
  uint64_t* acc_full = obs_bar + 1;
  uint64_t* act_lo = acc_full + 1;  // next operand tile, K-chunks 0-1 (columns 0..127) written
  uint64_t* act_hi = act_lo + 1;    // K-chunks 2-3 written
  uint64_t* act_rdy = act_lo;       // WIDE: [4] K-chunk pairs 0..3 of the next operand tile written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(act_lo + 4);
  float* ls_s = reinterpret_cast<float*>(bars + (WIDE ? 32 : 16));  // log_std[32], exp(log_std)[32]
  float* sig_s = ls_s + 32;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = a.L, T = a.T;
  const int m0 = blockIdx.x * kRows;

  if (threadIdx.x == 0) {
    for (int s = 0; s < (WIDE ? P.nstages : kStages); ++s) {
      ptx::mbar_init(&wfull[s], 1);
      ptx::mbar_init(&wempty[s], 1);
    }
    ptx::mbar_init(obs_bar, 1);
    ptx::mbar_init(acc_full, 1);
    for (int p = 0; p < (WIDE ? 4 : 2); ++p) ptx::mbar_init(&act_rdy[p], kEpiWarps);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&a.map_obs);
    for (int l = 0; l <= L; ++l) ptx::tma_prefetch_desc(&a.map_w[l]);
  }
  // two 256-column accumulators: layer l+1's MMAs run while layer l's epilogue drains
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
      const int nobs = (a.S_p + 63) / 64;
      ptx::mbar_arrive_expect_tx(obs_bar, nobs * kChunk);
      for (int kc = 0; kc < nobs; ++kc) ptx::tma_load_2d(act_buf0 + kc * kChunk, &a.map_obs, obs_bar, kc * 64, m0);
      int it = 0;
      for (int t = 0; t < T && WIDE; ++t)
        for (int l = 0; l <= L; ++l) {  // one [<=128 rows x 64 K] box per (K-chunk, N part)
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
      for (int t = 0; t < T && !WIDE; ++t)
        for (int l = 0; l <= L; ++l) {
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
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0 && WIDE) {
      ptx::mbar_wait_sleep(obs_bar, 0);
      int it = 0;
      uint32_t ph[4] = {0u, 0u, 0u, 0u};
      for (int t = 0; t < T; ++t)
        for (int l = 0; l <= L; ++l) {
          const bool first = t == 0 && l == 0;
          const int K = a.in_p[l], nk = (K + 63) / 64, N = a.out_n[l], np = (N + 127) / 128;
          const uint32_t in = ptx::smem_u32(smem + P.in_off[l]);
          const uint32_t acc = tmem + uint32_t(P.tmem[l]);
          int ready = 0;  // input K-chunk pairs known written
          if (!first && P.drain[l])  // accumulator overlaps the previous layer's: wait for its whole drain
            for (; ready < (nk + 1) / 2; ++ready) ptx::mbar_wait(&act_rdy[ready], (ph[ready]++) & 1);
          for (int kc = 0; kc < nk; ++kc) {
            if (!first && (kc >> 1) == ready) {
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
              for (int k = 0; k < ks; ++k) {
                const uint64_t ad = ptx::umma_desc_sw128(in + kc * kChunk + k * 32, 16, 1024);
                const uint64_t bd = ptx::umma_desc_sw128(wb + k * 32, 16, 1024);
                ptx::mma_bf16(acc + p * 128, ad, bd, idesc, (kc > 0 || k > 0) ? 1u : 0u);
              }
              ptx::mma_commit(&wempty[s]);
            }
          }
          ptx::mma_commit(acc_full);
        }
    }
    if (lane == 0 && !WIDE) {
      ptx::mbar_wait_sleep(obs_bar, 0);
      int it = 0, ph_lo = 0, ph_hi = 0, acc_ph = 0;
      for (int t = 0; t < T; ++t)
        for (int l = 0; l <= L; ++l, ++acc_ph) {
          const bool first = t == 0 && l == 0;
          const uint32_t acc = tmem + (acc_ph & 1) * 256;
          const uint32_t idesc = ptx::umma_idesc_bf16(kRows, uint32_t(a.out_n[l]), 0, 0);
          const uint32_t in = ptx::smem_u32((l & 1) ? act_buf1 : act_buf0);
          const int K = a.in_p[l];
          const int nk = (K + 63) / 64;
          for (int kc = 0; kc < nk; ++kc, ++it) {
            if (!first && kc == 0) ptx::mbar_wait(act_lo, (ph_lo++) & 1);
            if (!first && kc == 2) ptx::mbar_wait(act_hi, (ph_hi++) & 1);
            const int s = it % kStages;
            ptx::mbar_wait(&wfull[s], (it / kStages) & 1);
            ptx::tc_fence_after();
            const uint32_t wb = ptx::smem_u32(wring + s * kWStage);
            const int ks = min(4, (K - kc * 64 + 15) / 16);
            for (int k = 0; k < ks; ++k) {
              const uint64_t ad = ptx::umma_desc_sw128(in + kc * kChunk + k * 32, 16, 1024);
              const uint64_t bd = ptx::umma_desc_sw128(wb + k * 32, 16, 1024);
              ptx::mma_bf16(acc, ad, bd, idesc, (kc > 0 || k > 0) ? 1u : 0u);
            }
            ptx::mma_commit(&wempty[s]);
          }
          if (!first && nk <= 2) ptx::mbar_wait(act_hi, (ph_hi++) & 1);  // keep the phases paired
          ptx::mma_commit(acc_full);
        }
    }
  } else {
    // ------------------------------------------------ epilogue + env threads
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const int h = (warp - 2) >> 2;    // column group 0..3
    const int row = q * 32 + lane;    // accumulator row of this thread
    const int tid = threadIdx.x - 64;  // 0..511
    const int el = tid >> 2, sub = tid & 3;
    const int env = m0 + el;
    const bool valid = env < a.N;
    const int gid = a.env0 + env;
    const int A = a.A, S = a.S, S_p = a.S_p;
    int st = 0, len = 1, cnt = 0;
    float xs[MAXB][4];  // env state, register-resident for the whole rollout
#pragma unroll
    for (int bi = 0; bi < MAXB; ++bi)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = (sub + 4 * bi) * 4 + j;
        xs[bi][j] = valid && i < S ? a.x[(long long)env * S + i] : 0.f;
      }
    if (valid) {
      st = a.ep_step[env];
      len = a.ep_len[env];
      cnt = a.ep_count[env];
    }
    const uint32_t it0 = uint32_t(a.ctl->iteration) * uint32_t(T);
    if (tid < A) {  // first read after the first epi_bar (head phase of step 0)
      const float ls = a.log_std[tid];
      ls_s[tid] = ls;
      sig_s[tid] = expf(ls);
    }
    int accph = 0;
    for (int t = 0; t < T; ++t) {
      // ---- hidden layers: bias + ELU -> bf16 operand tile of the next layer
      for (int l = 0; l < L; ++l) {
        const uint32_t acc = WIDE ? tmem + uint32_t(P.tmem[l]) : tmem + (accph & 1) * 256;
        ptx::mbar_wait_sleep(acc_full, accph & 1);
        ++accph;
        ptx::tc_fence_after();
        trace_at(a, t * 16 + 2 * l);
        uint8_t* out = WIDE ? smem + P.in_off[l + 1] : (l & 1) ? act_buf0 : act_buf1;
        const float* bias = a.bias[l];
        const int nchunks = a.out_n[l] / 32;
        // pass 0: columns 0..127 (chunks h), then release K-chunks 0-1 to the next layer's MMA;
        // pass 1: columns 128..255 (chunks h + 4), then release K-chunks 2-3 (WIDE: up to 4 passes).
        const int npass = WIDE ? (a.out_n[l] + 127) / 128 : 2;
#pragma unroll 1
        for (int pass = 0; pass < npass; ++pass) {
          const int c = h + 4 * pass;
          if (c < nchunks) {
          uint32_t r[32];
          ptx::tmem_ld_32x32b_x32(acc + (static_cast<uint32_t>(q * 32) << 16) + c * 32, r);
          ptx::tmem_ld_wait();
          const float4* b4 = reinterpret_cast<const float4*>(bias + c * 32);
          uint32_t packed[16];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 b = __ldg(b4 + j);
            const float2 y0 = bias_elu2(make_float2(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1])),
                                        make_float2(b.x, b.y));
            const float2 y1 = bias_elu2(make_float2(__uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])),
                                        make_float2(b.z, b.w));
            packed[2 * j] = pack_bf16(y0.x, y0.y);
            packed[2 * j + 1] = pack_bf16(y1.x, y1.y);
          }
          uint8_t* chunk = out + (c >> 1) * kChunk + row * 128;
          const int u0 = (c & 1) * 4;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4*>(chunk + (((u0 + j) ^ (row & 7)) << 4)) =
                make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]);
          }
          ptx::fence_proxy_async_smem();
          ptx::tc_fence_before();
          __syncwarp();
          if (pass == npass - 1) trace_at(a, t * 16 + 2 * l + 1);
          if (lane == 0) ptx::mbar_arrive(WIDE ? &act_rdy[pass] : pass == 0 ? act_lo : act_hi);
        }
      }

      // ---- policy head: mu = acc + b_mu into smem (aliases the head's input tile)
      const uint32_t hacc = WIDE ? tmem + uint32_t(P.tmem[L]) : tmem + (accph & 1) * 256;
      ptx::mbar_wait_sleep(acc_full, accph & 1);
      ++accph;
      ptx::tc_fence_after();
      trace_at(a, t * 16 + 10);
      float* mu_s = reinterpret_cast<float*>(WIDE ? smem + P.in_off[L] : (L & 1) ? act_buf1 : act_buf0);
      float* u_s = mu_s + kRows * kMuLd;
      if (h == 0) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(hacc + (static_cast<uint32_t>(q * 32) << 16), r);
        ptx::tmem_ld_wait();
        for (int i = 0; i < A; ++i) mu_s[row * kMuLd + i] = __uint_as_float(r[i]) + a.bias[L][i];
      }
      ptx::tc_fence_before();
      epi_bar();

      // ---- actions: work item w = (Philox block w / 2, Box-Muller pair w % 2) -> actions
      // 4 (w / 2) + 2 (w % 2) + {0, 1}; thread `sub` of env `el` takes items sub, sub + 4, ...
      // The dynamics only need tanh(clip(a)), so it is computed once per action here.
      const uint32_t step = it0 + uint32_t(t);
      float lp_part = 0.f, usq_part = 0.f;
      if (valid) {
        for (int w = sub; w < 2 * ((A + 3) / 4); w += 4) {
          const int blk = w >> 1, p = w & 1;
          uint32_t rr[4];
          rng::draw(a.seed, uint32_t(gid), step, uint32_t(blk), rng::kNoise, rr);
          const uint32_t r0 = p ? rr[2] : rr[0], r1 = p ? rr[3] : rr[1];  // no dynamic indexing
          const float rad = sqrtf(-2.0f * logf(rng::u01_open0(r0)));
          const float th = kTwoPi * rng::u01(r1);
          float sn, cs;
          sincosf(th, &sn, &cs);
          const float nrm[2] = {rad * cs, rad * sn};
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int ai = blk * 4 + 2 * p + j;
            if (ai < A) {
              const float mu = mu_s[el * kMuLd + ai];
              const float ls = ls_s[ai], sig = sig_s[ai];
              const float act = mu + sig * nrm[j];
              const float z = (act - mu) / sig;
              lp_part += -0.5f * z * z - ls - kLog2PiHalf;
              const float u = fminf(fmaxf(act, -1.f), 1.f);
              usq_part += u * u;
              u_s[el * kMuLd + ai] = tanhf(u);
              a.act[((long long)t * a.N + env) * A + ai] = act;
            }
          }
        }
      }
      lp_part += __shfl_xor_sync(0xffffffffu, lp_part, 1);
      lp_part += __shfl_xor_sync(0xffffffffu, lp_part, 2);
      usq_part += __shfl_xor_sync(0xffffffffu, usq_part, 1);
      usq_part += __shfl_xor_sync(0xffffffffu, usq_part, 2);
      __syncwarp();
      trace_at(a, t * 16 + 11);

      // ---- dynamics on the register-resident state: thread `sub` owns dim blocks
      // k = sub + 4 bi (4 dims each); the right neighbour of a block's last dim is the
      // first dim of block k + 1 (thread (sub + 1) & 3) or, past dim S - 1, dim 0.
      const int base = lane & ~3, nxt = base + ((sub + 1) & 3);
      const float x0 = __shfl_sync(0xffffffffu, xs[0][0], base);
      float xn[MAXB][4];
      float xsq_part = 0.f;
#pragma unroll
      for (int bi = 0; bi < MAXB; ++bi) {
        const float nA = __shfl_sync(0xffffffffu, xs[bi][0], nxt);
        const float nB = __shfl_sync(0xffffffffu, xs[bi + 1 < MAXB ? bi + 1 : bi][0], nxt);
        const int blk = sub + 4 * bi;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = blk * 4 + j;
          xn[bi][j] = 0.f;
          if (valid && i < S) {
            const float nb = i + 1 >= S ? x0 : j < 3 ? xs[bi][j + 1] : (sub == 3 ? nB : nA);
            const float drive = u_s[el * kMuLd + i % A];  // tanh(clip(a)), see above
            const float xi = xs[bi][j];
            const float inner = __fadd_rn(__fsub_rn(drive, __fmul_rn(kDamp, xi)), __fmul_rn(kCouple, env_sin(nb)));
            xn[bi][j] = __fadd_rn(xi, __fmul_rn(kDt, inner));
            xsq_part = __fadd_rn(xsq_part, __fmul_rn(xn[bi][j], xn[bi][j]));
          }
        }
      }
      xsq_part += __shfl_xor_sync(0xffffffffu, xsq_part, 1);
      xsq_part += __shfl_xor_sync(0xffffffffu, xsq_part, 2);
      const float xn0 = __shfl_sync(0xffffffffu, xn[0][0], base);
      const bool done = st + 1 >= len;
      const int count = cnt + (done ? 1 : 0);
      __nv_bfloat16* xo = a.X_roll + ((long long)(t + 1) * a.N + env) * S_p;
#pragma unroll
      for (int bi = 0; bi < MAXB; ++bi) {
        const int blk = sub + 4 * bi;
        if (valid && blk * 4 < S_p) {
          uint32_t rr[4] = {0u, 0u, 0u, 0u};
          if (done && blk * 4 < S) rng::draw(a.seed, uint32_t(gid), uint32_t(count), uint32_t(blk), rng::kReset, rr);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int i = blk * 4 + j;
            xs[bi][j] = i >= S ? 0.f : done ? __fsub_rn(__fmul_rn(rng::u01(rr[j]), 0.2f), 0.1f) : xn[bi][j];
          }
          // 4 bf16 (8 bytes) of the next observation row: HBM rollout buffer (pads = 0)
          const uint2 pk = make_uint2(pack_bf16(xs[bi][0], xs[bi][1]), pack_bf16(xs[bi][2], xs[bi][3]));
          *reinterpret_cast<uint2*>(xo + blk * 4) = pk;
        }
      }
      if (valid) {
        if (sub == 0) {
          const long long o = (long long)t * a.N + env;
          const float r0 = __fsub_rn(__fadd_rn(1.0f, xn0), __fdiv_rn(__fmul_rn(kCtrl, usq_part), float(A)));
          a.rew[o] = __fsub_rn(r0, __fdiv_rn(__fmul_rn(kStateC, xsq_part), float(S)));
          a.logp[o] = lp_part;
          a.done[o] = done ? 1 : 0;
        }
        st = done ? 0 : st + 1;
        cnt = count;
      }

      // ---- next observation into the layer-0 operand tile (pads written as zero)
      trace_at(a, t * 16 + 12);
      epi_bar();  // mu / u staging may alias the obs tile
      if (t + 1 < T) {
        if (valid) {
#pragma unroll
          for (int bi = 0; bi < MAXB; ++bi) {
            const int blk = sub + 4 * bi;
            if (blk * 4 < S_p) {
              const uint2 pk = make_uint2(pack_bf16(xs[bi][0], xs[bi][1]), pack_bf16(xs[bi][2], xs[bi][3]));
              *reinterpret_cast<uint2*>(act_buf0 + (blk >> 4) * kChunk + sw128(el, blk * 4)) = pk;
            }
          }
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        trace_at(a, t * 16 + 13);
        if (lane == 0) {
          if constexpr (WIDE) {
            for (int p = 0; p < (S_p + 127) / 128; ++p) ptx::mbar_arrive(&act_rdy[p]);
          } else {
            ptx::mbar_arrive(act_lo);
            ptx::mbar_arrive(act_hi);
          }
        }
      }
    }
    if (valid) {
      if (sub == 0) {
        a.ep_step[env] = st;
        a.ep_count[env] = cnt;
      }
#pragma unroll
      for (int bi = 0; bi < MAXB; ++bi)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = (sub + 4 * bi) * 4 + j;
          if (i < S) a.x[(long long)env * S + i] = xs[bi][j];
        }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

}  // namespace

bool rollout_fusable(int L, const int* widths_p, int S_p, int A) {
  if (L < 1 || L > kRollMaxL || S_p > 128 || A > 31 || A < 1) return false;
  for (int l = 1; l <= L; ++l)
    if (widths_p[l] > 256 || widths_p[l] % 32) return false;
  // the mu / u staging must fit in one operand tile
  return 2 * kRows * kMuLd * 4 <= int(kActBytes);
}

bool plan_wide(int L, const int* widths_p, int head_n, bool rollout, WidePlan* out) {
  if (L < 1 || L > kRollMaxL) return false;
  WidePlan P{};
  auto chunks = [](int w) { return (w + 63) / 64; };
  int main = 0;  // K-chunks of the in-place activation region
  for (int l = 0; l <= L; ++l) {
    if (widths_p[l] <= 0 || widths_p[l] > 512 || widths_p[l] % 32) return false;
    if (l > 0) main = std::max(main, chunks(widths_p[l]));
  }
  const int obs = chunks(widths_p[0]);
  const uint32_t budget = 232448u - 512u - 1024u;  // dynamic smem - barriers - alignment slack
  if (rollout) {  // obs written in place by the env threads; mu / tanh(u) staging [2][128][kMuLd]
    main = std::max({main, obs, int((2 * kRows * kMuLd * 4 + kChunk - 1) / kChunk)});
  } else {  // own observation buffer when 4 ring stages still fit beside it (next tile's load overlaps)
    P.obs_sep = uint32_t(main + obs) * kChunk + 4 * kWideStage <= budget;
    if (!P.obs_sep) main = std::max(main, obs);
  }
  P.in_off[0] = P.obs_sep ? uint32_t(main) * kChunk : 0u;
  P.ring_off = uint32_t(main + (P.obs_sep ? obs : 0)) * kChunk;
  if (P.ring_off + 2 * kWideStage > budget) return false;
  P.nstages = std::min<int>(8, int((budget - P.ring_off) / kWideStage));
  P.bar_off = P.ring_off + uint32_t(P.nstages) * kWideStage;
  P.smem = P.bar_off + 512 + 1024;
  int prev_lo = 0, prev_hi = 0;
  for (int l = 0; l <= L; ++l) {
    const int o = l < L ? widths_p[l + 1] : head_n;
    P.wrows[l] = std::min(128, o);
    if (l == 0) {
      P.tmem[0] = 0;
    } else if (prev_hi + o <= 512) {  // beside the previous accumulator
      P.tmem[l] = prev_hi;
    } else {  // from column 0: overlaps it unless it ends below the previous start
      P.tmem[l] = 0;
      P.drain[l] = o > prev_lo;
    }
    prev_lo = P.tmem[l];
    prev_hi = P.tmem[l] + o;
  }
  P.wrap = P.tmem[L] < widths_p[1];
  *out = P;
  return true;
}

bool rollout_wide_fusable(int L, const int* widths_p, int S_p, int A, WidePlan* plan) {
  if (L < 1 || L > kRollMaxL || S_p > 128 || A > 31 || A < 1) return false;
  return plan_wide(L, widths_p, A <= 16 ? 16 : 32, true, plan);  // obs / mu in the in-place region
}

template <int MAXB, bool WIDE>
void launch_t(const RolloutArgs& a, cudaStream_t s) {
  static bool configured = false;
  const uint32_t smem = WIDE ? a.plan.smem : kSmemBytes;
  if (!configured) {
    GMI_CUDA_CHECK(
        cudaFuncSetAttribute(rollout_kernel<MAXB, WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    configured = true;
  }
  const int blocks = (a.N + kRows - 1) / kRows;
  launch_pdl(rollout_kernel<MAXB, WIDE>, dim3(blocks), dim3(kThreads), smem, s, a);
}

void launch_rollout(const RolloutArgs& a, cudaStream_t s) {
  if (a.wide)
    launch_t<8, true>(a, s);
  else if (a.S_p <= 64)
    launch_t<4, false>(a, s);
  else
    launch_t<8, false>(a, s);
}

}  // namespace gmi::ppo
