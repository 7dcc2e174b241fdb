// Persistent, warp-specialised tcgen05 GEMM for the actor-critic MLP layers (sm_100a).
//
//   D[m][n] = sum_k A(m,k) * B(n,k)        bf16 operands, fp32 accumulation in TMEM
//
// One CTA per SM walks a static tile schedule (grouped problems x split-K slabs x M x N
// tiles). Warp 0 streams operands with TMA (128B swizzle) through a STAGES-deep
// shared-memory ring; warp 1 issues tcgen05.mma (M = 128, N = BN, K = 16) into one of two
// TMEM accumulators; the epilogue warps drain the other accumulator concurrently
// (tcgen05.ld -> fused epilogue -> swizzled smem staging -> TMA store), so the epilogue
// of tile i overlaps the MMAs of tile i+1. Either operand may be K-major (row-major
// [rows x K]) or MN-major (row-major [K x rows]); MN-major lets the weight-gradient GEMM
// (dW = dPre^T H, reduction over minibatch rows) read activations in place.
//
// Weight-stationary mode (WS = 1: N <= BN, K <= 256; WS = 2: N <= BN <= 128, K <= 512; no
// split-K): each CTA serves one
// problem (CTA index mod problems), loads that problem's whole B operand (the layer's
// weights, <= 128 KB) into shared memory once and then streams only the A tiles
// (activations / dPre rows). This removes the per-tile weight re-reads that made the
// training-forward and input-gradient GEMMs L2-bandwidth-bound.
//
// Epilogues:
//   EPI_BIAS_ELU  hidden-layer forward: bf16 out = elu(acc + bias[n])
//   EPI_DACT      hidden-layer backward: bf16 out = acc * elu'(H[m][n]), elu' = H > 0 ? 1 : H + 1
//   EPI_F32       fp32 [split][m][n] (split-K weight-gradient slabs, head outputs)
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

#include "gemm_types.hpp"
#include "launch.cuh"
#include "ptx.cuh"

namespace gmi {

// elu on a pair, (acc + bias) -> x > 0 ? x : expm1(x), in 1.5 FMA-pipe instructions, one
// SFU exp and two min/max per element (the epilogue is issue-bound, so this is what sets
// the GEMM's speed at K <= 256). n = 2^(x log2 e) - 1 has absolute error ~1e-7
// (ex2.approx), i.e. well below bf16 output rounding except at |x| < ~1e-3, where
// max(min(n, 0), x) picks whichever of n and x is closer to expm1(x) (expm1(x) >= x).
__device__ __forceinline__ float2 bias_elu2(float2 acc, float2 bias) {
  const float2 x = ptx::add2(acc, bias);
  const float2 t = ptx::mul2(x, make_float2(1.4426950408889634f, 1.4426950408889634f));
  const float2 n = ptx::add2(make_float2(ptx::ex2_approx(t.x), ptx::ex2_approx(t.y)), make_float2(-1.f, -1.f));
  return make_float2(fmaxf(fminf(n.x, 0.f), x.x), fmaxf(fminf(n.y, 0.f), x.y));
}

// dPre = dH * elu'(H), elu'(H) = H > 0 ? 1 : H + 1 (H = elu output). acc * (min(H,0) + 1)
// equals fma(acc, min(H,0), acc) exactly (min(H,0) + 1 is exact for bf16 H >= -1), so the
// packed FFMA2 form is bit-identical to the scalar definition.
__device__ __forceinline__ float2 dact2(float2 acc, uint32_t h2) {
  const float2 h = make_float2(__uint_as_float(h2 << 16), __uint_as_float(h2 & 0xFFFF0000u));
  return ptx::fma2(acc, make_float2(fminf(h.x, 0.f), fminf(h.y, 0.f)), acc);
}

// n / d for 0 <= n < 2^24, d >= 1 via an fp32 reciprocal (exact after one correction step);
// the tile decode runs on every warp once per tile, so integer division is worth avoiding.
__device__ __forceinline__ int fdiv(int n, int d, float rd) {
  int q = __float2int_rz(__int2float_rn(n) * rd);
  const int r = n - q * d;
  q += (r >= d) - (r < 0);
  return q;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Development trace (tools/gemm_trace.py): compiled in only with `make TRACE=1` (-DGMI_TRACE).
__device__ __forceinline__ void gemm_stamp(unsigned long long* tr, int lt, int k) {
#ifdef GMI_TRACE
  if (tr && blockIdx.x == 0 && lt < 8) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[lt * 16 + k] = t;
  }
#else
  (void)tr, (void)lt, (void)k;
#endif
}

#ifndef GMI_WS_STAGES
#define GMI_WS_STAGES 8
#endif
#ifndef GMI_WS_STAGING
#define GMI_WS_STAGING 1
#endif
#ifndef GMI_DX_AUX_BUFS
#define GMI_DX_AUX_BUFS 2
#endif

template <int BN, int EPI, int WS>
struct GemmSmem {
  static constexpr int kEpiWarps = gemm_epi_warps(EPI);
  // WS: single epilogue staging buffer per warp (2 stages + double staging measured 3% slower
  // on B200: the A ring starves the MMA)
  static constexpr uint32_t kA = kGemmBlockM * kGemmBlockK * 2;  // 16 KB
  static constexpr uint32_t kB = BN * kGemmBlockK * 2;           // one k-block of B
  static constexpr uint32_t kBRes = WS ? gemm_ws_kb(WS) * kB : 0;  // resident B (WS)
  // split-K fp32 slabs at BN = 256 (one tile per CTA): a 4th operand stage beats double
  // staging of the once-per-CTA epilogue (weight-gradient phase 0.99 -> 0.96 ms per iteration)
  static constexpr bool kDw4 = !WS && EPI == 2;  // every split-K launch: one tile per CTA
  static constexpr int kStagingBufs = WS || kDw4 ? GMI_WS_STAGING : 2;
  static constexpr uint32_t kStaging = EPI == 2 ? 4096 : 2048;  // one 32x32 chunk per warp
  // WS: as many activation stages as fit next to the resident weights, up to two whole tiles
  // (K <= 256 is 4 k-blocks), so the next tile's rows are in flight while this tile's MMAs run
  // WS forward: the CTA's bias row (one problem per CTA, n0 = 0) staged in shared memory once
  static constexpr uint32_t kBias = (WS && EPI == 0) ? BN * 4 : 0;
  // WS input gradient: the elu' operand (H rows of the tile) staged by TMA, double-buffered
  // [buf][BN / 64 boxes][128 rows][64 cols] SW128, instead of per-thread global loads in the epilogue
  // (BN <= 128: at BN = 256 the resident weights leave no room; the global-load path is kept)
  // (WS = 2: the 128 KB of resident weights leave no room either)
  static constexpr int kAuxBufs = (WS == 1 && EPI == 1 && BN <= 128) ? GMI_DX_AUX_BUFS : 0;
  static constexpr uint32_t kAuxBox = kGemmBlockM * 128;  // 128 rows x 64 bf16 columns
  static constexpr uint32_t kAux = kAuxBufs * (BN / 64) * kAuxBox;
  static constexpr int kWsFit = int((232448u - 1536u - kBias - kAux - kBRes - kEpiWarps * kStagingBufs * kStaging) / kA);
  // split-K weight gradients: as many operand stages as fit (up to 8) -- the kernel streams a
  // long K range per CTA and is bound by bytes in flight
  static constexpr int kDwFit = int((232448u - 1536u - kEpiWarps * kStagingBufs * kStaging) / (kA + kB));
  static constexpr int kStages = WS     ? (kWsFit < GMI_WS_STAGES ? kWsFit : GMI_WS_STAGES)
                                 : kDw4 ? (kDwFit < 8 ? kDwFit : 8)
                                        : (BN == 256 ? 3 : 4);
  static constexpr uint32_t kStage = WS ? kA : kA + kB;
  static constexpr uint32_t kAuxOff = kStages * kStage + kBRes;  // 1024-aligned (SW128 boxes)
  static constexpr uint32_t kBarOff = kAuxOff + kAux + kEpiWarps * kStagingBufs * kStaging + kBias;
  static constexpr uint32_t kBytes = kBarOff + 512 + 1024;  // + barriers + alignment slack
  static constexpr uint32_t kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
  static_assert(kBytes <= 232448, "shared memory budget");
};

// Total tiles of a weight-stationary launch (one problem per CTA, splits == 1, N <= BN).
__device__ __forceinline__ int ntile_total_ws(const GemmParams& P) {
  return (P.prob[0].M + kGemmBlockM - 1) / kGemmBlockM * P.num_problems;
}

// CS = 1 (EPI_F32 with MN-major A only): 4 extra warps sum the A stages over K (bias gradient).
template <int BN, int A_MN, int B_MN, int EPI, int WS, int CS = 0>
__global__ void __launch_bounds__(gemm_threads(EPI) + 128 * CS, 1)
    gemm_tcgen05_kernel(const __grid_constant__ GemmParams P) {
  using L = GemmSmem<BN, EPI, WS>;
  constexpr int S = L::kStages;
  constexpr int kEpiWarps = L::kEpiWarps;
  constexpr uint32_t kIdesc = ptx::umma_idesc_bf16(kGemmBlockM, BN, A_MN, B_MN);
  static_assert(BN % 64 == 0 && BN <= 256, "BN must be 64, 128 or 256");
  static_assert(!CS || (EPI == EPI_F32 && A_MN && !WS), "column sums: split-K weight gradient only");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::align_smem_1024(smem_raw);
  uint8_t* b_res = smem + S * L::kStage;  // WS: resident B, k-block j at j * kB
  uint8_t* aux_s = smem + L::kAuxOff;     // WS input gradient: staged elu' operand
  uint8_t* staging = aux_s + L::kAux;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;   // [2] accumulator ready
  uint64_t* tempty_bar = tfull_bar + 2;  // [2] accumulator drained
  uint64_t* bres_bar = tempty_bar + 2;   // WS: resident B landed
  uint64_t* bfree_bar = bres_bar + 1;    // chained WS: every MMA on the resident B done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfree_bar + 1);
  // chained WS: per epilogue warp, how many of the CTA's tiles (in processing order, all
  // layers) have their H stores complete in global memory
  volatile int* stored_s = reinterpret_cast<volatile int*>(tmem_slot + 1);
  uint64_t* auxf_bar = reinterpret_cast<uint64_t*>(smem + L::kBarOff + 256);  // [kAuxBufs] aux landed
  uint64_t* auxe_bar = auxf_bar + 2;                                          // [kAuxBufs] aux consumed

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const GemmProblem& p0 = P.prob[0];
  auto load_b = [&](const GemmProblem& pr, uint8_t* sb, uint64_t* bar, int n0, int k0) {
    if constexpr (B_MN) {
#pragma unroll
      for (int j = 0; j < BN / 64; ++j) ptx::tma_load_2d(sb + j * 8192, &pr.map_b, bar, n0 + 64 * j, k0 + pr.b_row0);
    } else {
      ptx::tma_load_2d(sb, &pr.map_b, bar, k0, n0 + pr.b_row0);
    }
  };
  // chained layers (WS forward only): layer c's problems are prob[c * num_problems + i]
  const int nchain = (WS && EPI == EPI_BIAS_ELU && P.chain > 1) ? P.chain : 1;
  const int mtiles = (p0.M + kGemmBlockM - 1) / kGemmBlockM;
  const int ntiles = (p0.N + BN - 1) / BN;
  const int per_prob = P.splits * mtiles * ntiles;
  const int ntile_total = P.hetero ? P.tile0[P.num_problems] : per_prob * P.num_problems;
  const int nkb_total = (p0.K + kGemmBlockK - 1) / kGemmBlockK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1 + 4 * CS);  // MMA commit (+ 4 column-sum warps)
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull_bar[b], 1);
      ptx::mbar_init(&tempty_bar[b], kEpiWarps);
    }
    ptx::mbar_init(bres_bar, 1);
    ptx::mbar_init(bfree_bar, 1);
    for (int b = 0; b < L::kAuxBufs; ++b) {
      ptx::mbar_init(&auxf_bar[b], 1);
      ptx::mbar_init(&auxe_bar[b], kEpiWarps);
    }
    for (int e = 0; e < kEpiWarps; ++e) stored_s[e] = 0;
    ptx::fence_mbar_init();
    for (int i = 0; i < P.num_problems * nchain; ++i) {
      ptx::tma_prefetch_desc(&P.prob[i].map_a);
      ptx::tma_prefetch_desc(&P.prob[i].map_b);
      ptx::tma_prefetch_desc(&P.prob[i].map_out);
      if constexpr (L::kAuxBufs > 0) ptx::tma_prefetch_desc(&P.prob[i].map_aux);
    }
    if constexpr (WS) {
      // stable weights: the whole resident B before griddepcontrol.wait (overlaps the tail of
      // the previous kernel); the CTA's problem is blockIdx.x % problems for every tile
      if (P.b_stable && int(blockIdx.x) < ntile_total_ws(P)) {
        const GemmProblem& pb = P.prob[blockIdx.x % P.num_problems];
        const int nkb = (pb.K + kGemmBlockK - 1) / kGemmBlockK;
        ptx::mbar_arrive_expect_tx(bres_bar, uint32_t(nkb) * L::kB);
        for (int i = 0; i < nkb; ++i) load_b(pb, b_res + i * L::kB, bres_bar, 0, i * kGemmBlockK);
      }
    }
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, L::kTmemCols);
  pdl_trigger();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // operands / bias / aux come from the preceding kernels in the stream

  const int mn_tiles = mtiles * ntiles;
  const float r_per_prob = 1.f / float(per_prob), r_mn = 1.f / float(mn_tiles), r_n = 1.f / float(ntiles);
  const float r_np = 1.f / float(P.num_problems);
  auto decode = [&](int tile, int& prob, int& split, int& m0, int& n0, int& kb0, int& nkb) {
    if constexpr (WS) {  // tile = m_tile * problems + prob; gridDim.x % problems == 0
      const int mt = fdiv(tile, P.num_problems, r_np);
      prob = tile - mt * P.num_problems;
      split = 0;
      m0 = mt * kGemmBlockM;
      n0 = 0;
      kb0 = 0;
      nkb = nkb_total;
      return;
    }
    if (P.hetero) {  // problem-own tile counts: find the problem, then split / m / n inside it
      prob = 0;
      while (prob + 1 < P.num_problems && tile >= P.tile0[prob + 1]) ++prob;
      const GemmProblem& pp = P.prob[prob];
      const int nt = (pp.N + BN - 1) / BN, mn = ((pp.M + kGemmBlockM - 1) / kGemmBlockM) * nt;
      int r = tile - P.tile0[prob];
      split = r / mn;
      r -= split * mn;
      const int mt = r / nt;
      m0 = mt * kGemmBlockM;
      n0 = (r - mt * nt) * BN;
    } else {
      prob = fdiv(tile, per_prob, r_per_prob);
      int r = tile - prob * per_prob;
      split = fdiv(r, mn_tiles, r_mn);
      r -= split * mn_tiles;
      const int mt = fdiv(r, ntiles, r_n);
      m0 = mt * kGemmBlockM;
      n0 = (r - mt * ntiles) * BN;
    }
    kb0 = split * P.prob[prob].kb_per_split;
    const int kb1 = min(nkb_total, kb0 + P.prob[prob].kb_per_split);
    nkb = kb1 > kb0 ? kb1 - kb0 : 0;
  };

  if (warp == 0) {
    // ---------------- TMA producer (one lane)
    if (lane == 0) {
      int it = 0, plt = 0;
      const int ntl = (ntile_total - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x);  // tiles per layer
      for (int ci = 0; ci < nchain; ++ci) {
      const int pb0 = ci * P.num_problems;
      int lt = 0;
      for (int tile = blockIdx.x; tile < ntile_total; tile += gridDim.x, ++plt, ++lt) {
        int prob, split, m0, n0, kb0, nkb;
        decode(tile, prob, split, m0, n0, kb0, nkb);
        const GemmProblem& pr = P.prob[pb0 + prob];
        if (nchain > 1) {
          nkb = (pr.K + kGemmBlockK - 1) / kGemmBlockK;
          if (ci > 0) {  // this row tile's layer ci-1 output (stored by this CTA) is in global memory
            const int need = (ci - 1) * ntl + lt + 1;
            for (int e = 0; e < kEpiWarps; ++e)
              while (stored_s[e] < need) __nanosleep(64);
            __threadfence_block();
            ptx::fence_proxy_async_global();
          }
        }
        gemm_stamp(P.trace, plt, 7);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % S;
          if (it >= S) ptx::mbar_wait(&empty_bar[s], ((it / S) - 1) & 1);
          uint8_t* sa = smem + s * L::kStage;
          const int k0 = (kb0 + i) * kGemmBlockK;
          // WS: the CTA's first tile also brings the resident B k-block i on the same barrier,
          // so the first MMAs start after one k-block instead of after the whole weight tile.
          const bool first_ws = WS && !P.b_stable && ci == 0 && it < nkb;
          ptx::mbar_arrive_expect_tx(&full_bar[s], L::kStage + (first_ws ? L::kB : 0u));
          if (first_ws) load_b(pr, b_res + i * L::kB, &full_bar[s], 0, k0);
          if constexpr (A_MN) {
#pragma unroll
            for (int j = 0; j < kGemmBlockM / 64; ++j)
              ptx::tma_load_2d(sa + j * 8192, &pr.map_a, &full_bar[s], m0 + 64 * j, k0 + pr.a_row0);
          } else {
            ptx::tma_load_2d(sa, &pr.map_a, &full_bar[s], k0, m0 + pr.a_row0);
          }
          if constexpr (!WS) load_b(pr, sa + L::kA, &full_bar[s], n0, k0);
        }
        if constexpr (L::kAuxBufs > 0) {  // the tile's elu' operand rows, into the aux ring
          const int ab = plt % L::kAuxBufs;
          if (plt >= L::kAuxBufs) ptx::mbar_wait(&auxe_bar[ab], ((plt / L::kAuxBufs) - 1) & 1);
          ptx::mbar_arrive_expect_tx(&auxf_bar[ab], (BN / 64) * L::kAuxBox);
#pragma unroll
          for (int j = 0; j < BN / 64; ++j)
            ptx::tma_load_2d(aux_s + (ab * (BN / 64) + j) * L::kAuxBox, &pr.map_aux, &auxf_bar[ab], n0 + 64 * j, m0);
        }
        if (ci > 0 && lt == 0) {  // the layer's resident weights, once every MMA on the previous ones is
          // done (after the first tile's activation loads, which only need free ring stages)
          ptx::mbar_wait(bfree_bar, (ci - 1) & 1);
          const GemmProblem& pb = P.prob[pb0 + blockIdx.x % P.num_problems];
          const int nkbb = (pb.K + kGemmBlockK - 1) / kGemmBlockK;
          ptx::mbar_arrive_expect_tx(bres_bar, uint32_t(nkbb) * L::kB);
          for (int i = 0; i < nkbb; ++i) load_b(pb, b_res + i * L::kB, bres_bar, 0, i * kGemmBlockK);
        }
        gemm_stamp(P.trace, plt, 8);
      }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one lane), double-buffered TMEM accumulators
    if (lane == 0) {
      int it = 0, lt = 0, bph = 0;
      if (WS && P.b_stable && int(blockIdx.x) < ntile_total) ptx::mbar_wait(bres_bar, (bph++) & 1);  // resident B landed
      for (int ci = 0; ci < nchain; ++ci) {
      if (ci > 0 && int(blockIdx.x) < ntile_total) ptx::mbar_wait(bres_bar, (bph++) & 1);  // next layer's B landed
      for (int tile = blockIdx.x; tile < ntile_total; tile += gridDim.x, ++lt) {
        int prob, split, m0, n0, kb0, nkb;
        decode(tile, prob, split, m0, n0, kb0, nkb);
        if (nchain > 1) nkb = (P.prob[ci * P.num_problems + prob].K + kGemmBlockK - 1) / kGemmBlockK;
        const int buf = lt & 1;
        gemm_stamp(P.trace, lt, 0);
        if (lt >= 2) ptx::mbar_wait(&tempty_bar[buf], ((lt >> 1) - 1) & 1);
        gemm_stamp(P.trace, lt, 1);
        ptx::tc_fence_after();
        const uint32_t acc = tmem_base + buf * BN;
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % S;
          ptx::mbar_wait(&full_bar[s], (it / S) & 1);
          if (i == 0) gemm_stamp(P.trace, lt, 2);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + s * L::kStage);
          const uint32_t sb = WS ? ptx::smem_u32(b_res + i * L::kB) : sa + L::kA;
#pragma unroll
          for (int k = 0; k < kGemmBlockK / 16; ++k) {
            // K-major: step 16 elements (32 B) inside the swizzle atom.
            // MN-major: step 16 rows = two 8-row core groups (2 x 1024 B).
            const uint64_t ad = A_MN ? ptx::umma_desc_sw128(sa + k * 2048, 8192, 1024)
                                     : ptx::umma_desc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? ptx::umma_desc_sw128(sb + k * 2048, 8192, 1024)
                                     : ptx::umma_desc_sw128(sb + k * 32, 16, 1024);
            ptx::mma_bf16(acc, ad, bd, kIdesc, (i > 0 || k > 0) ? 1u : 0u);
          }
          ptx::mma_commit(&empty_bar[s]);
        }
        ptx::mma_commit(&tfull_bar[buf]);
        gemm_stamp(P.trace, lt, 3);
      }
      if (ci + 1 < nchain) ptx::mma_commit(bfree_bar);  // the resident B may be replaced
      }
    }
  } else if (warp < 2 + kEpiWarps) {
    // ---------------- epilogue warps: TMEM lane quarter q, every W-th 32-column chunk
    constexpr int W = kEpiWarps / 4;  // warps per lane quarter
    const int e = warp - 2;
    const int q = warp & 3;
    const int h = e >> 2;
    constexpr int kChunks = BN / 32;
    uint8_t* stage_base = staging + e * L::kStagingBufs * L::kStaging;
    float* bias_s = reinterpret_cast<float*>(staging + kEpiWarps * L::kStagingBufs * L::kStaging);
    int sbuf = 0;
    int lt = 0;
    const int ntl = (ntile_total - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x);  // tiles per layer
    for (int ci = 0; ci < nchain; ++ci) {
    const int pb0 = ci * P.num_problems;
    if constexpr (L::kBias > 0) {  // WS: this CTA's problem is blockIdx.x % problems for every tile
      const GemmProblem& pb = P.prob[pb0 + blockIdx.x % P.num_problems];
      if (ci > 0) asm volatile("bar.sync 1, %0;" ::"r"(kEpiWarps * 32));  // layer ci-1's bias reads done
      for (int i = e * 32 + lane; i < BN; i += kEpiWarps * 32) bias_s[i] = i < pb.N ? pb.bias[i] : 0.f;
      asm volatile("bar.sync 1, %0;" ::"r"(kEpiWarps * 32));
    }
    for (int tile = blockIdx.x, tl = 0; tile < ntile_total; tile += gridDim.x, ++lt, ++tl) {
      int prob, split, m0, n0, kb0, nkb;
      decode(tile, prob, split, m0, n0, kb0, nkb);
      const GemmProblem& pr = P.prob[pb0 + prob];
      if (nchain > 1) nkb = (pr.K + kGemmBlockK - 1) / kGemmBlockK;
      const int buf = lt & 1;
      const int rbase = m0 + q * 32;
      const int row = rbase + lane;
      // EPI_DACT: the elu' operand (H rows, bf16) is fetched one chunk ahead so its HBM/L2
      // latency overlaps the accumulator wait and the previous chunk's math.
      uint4 hv[4] = {}, hn[4] = {};
      auto load_aux = [&](int c, uint4(&dst)[4]) {
        const int col0 = n0 + c * 32;
        if (c < kChunks && col0 < pr.N && row < pr.M) {
          const uint4* hp = reinterpret_cast<const uint4*>(pr.aux + (long long)row * pr.ld_aux + col0);
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) dst[qd] = hp[qd];
        }
      };
      if constexpr (EPI == EPI_DACT && L::kAuxBufs == 0) load_aux(h, hv);
      // staged elu' operand: this thread's row of chunk c (32 columns = 4 x 16 B, SW128 box c / 2)
      auto lds_aux = [&](int c, uint4(&dst)[4]) {
        const uint8_t* box = aux_s + ((lt % (L::kAuxBufs > 0 ? L::kAuxBufs : 1)) * (BN / 64) + (c >> 1)) * L::kAuxBox;
#pragma unroll
        for (int qd = 0; qd < 4; ++qd)
          dst[qd] = *reinterpret_cast<const uint4*>(box + (q * 32 + lane) * 128 + ((((c & 1) * 4 + qd) ^ (lane & 7)) << 4));
      };
      unsigned long long* etr = (warp == 2 && lane == 0) ? P.trace : nullptr;
      ptx::mbar_wait(&tfull_bar[buf], (lt >> 1) & 1);
      gemm_stamp(etr, lt, 4);
      ptx::tc_fence_after();
      if constexpr (L::kAuxBufs > 0) ptx::mbar_wait(&auxf_bar[lt % L::kAuxBufs], (lt / L::kAuxBufs) & 1);
      // 16-column units of chunks c = h, h + W, ...: the TMEM load of the next unit is issued
      // before this unit's math, and the staging buffer is claimed only after the math, so TMEM
      // latency and the previous TMA store overlap useful work (the epilogue is latency-bound
      // at K <= 256); x16 units keep two loads in flight within the register budget.
      constexpr int kUnits = 2 * ((kChunks + W - 1) / W);
      const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * BN;
      uint32_t rr[2][16];
      if (n0 + h * 32 < pr.N) ptx::tmem_ld_32x32b_x16(trow + h * 32, rr[0]);
#pragma unroll
      for (int i = 0; i < kUnits; ++i) {
        const int c = h + (i >> 1) * W, half = i & 1;
        const int col0 = n0 + c * 32;
        if (c >= kChunks || col0 >= pr.N) break;  // warp-uniform
        uint32_t(&r)[16] = rr[i & 1];
        if constexpr (EPI == EPI_DACT && L::kAuxBufs == 0) {
          if (half == 0) load_aux(c + W, hn);
        }
        if constexpr (EPI == EPI_DACT && L::kAuxBufs > 0) {
          if (half == 0) lds_aux(c, hv);
        }
        ptx::tmem_ld_wait();
        if (i + 1 < kUnits) {
          const int cn = h + ((i + 1) >> 1) * W;
          if (cn < kChunks && n0 + cn * 32 < pr.N) ptx::tmem_ld_32x32b_x16(trow + cn * 32 + ((i + 1) & 1) * 16, rr[(i + 1) & 1]);
        }
        if (nkb == 0) {
#pragma unroll
          for (int j = 0; j < 16; ++j) r[j] = 0u;
        }
        uint8_t* st = stage_base + sbuf * L::kStaging;
        if constexpr (EPI == EPI_F32) {
          if (half == 0) {
            if (lane == 0) ptx::bulk_wait_read<L::kStagingBufs - 1>();  // this staging buffer's last store has read it
            __syncwarp();
          }
          // 32 fp32 = 8 x 16 B per row; SWIZZLE_128B: chunk ^= row & 7
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4*>(st + lane * 128 + (((half * 4 + j) ^ (lane & 7)) << 4)) =
                make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
        } else {
          uint32_t packed[8];
          if constexpr (EPI == EPI_BIAS_ELU) {
            const float4* b4 = reinterpret_cast<const float4*>((L::kBias > 0 ? bias_s : pr.bias) + col0 + half * 16);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 b = L::kBias > 0 ? b4[j] : __ldg(b4 + j);
              const float2 y0 = bias_elu2(make_float2(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1])),
                                          make_float2(b.x, b.y));
              const float2 y1 = bias_elu2(make_float2(__uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])),
                                          make_float2(b.z, b.w));
              packed[2 * j] = pack_bf16(y0.x, y0.y);
              packed[2 * j + 1] = pack_bf16(y1.x, y1.y);
            }
          } else {  // EPI_DACT
#pragma unroll
            for (int qd = 0; qd < 2; ++qd) {
              const uint4 hq = half ? hv[2 + qd] : hv[qd];
              const uint32_t hw[4] = {hq.x, hq.y, hq.z, hq.w};
#pragma unroll
              for (int x = 0; x < 4; ++x) {
                const int j = qd * 8 + x * 2;
                const float2 d = dact2(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), hw[x]);
                packed[j / 2] = pack_bf16(d.x, d.y);
              }
            }
            if (half == 1 && L::kAuxBufs == 0) {
#pragma unroll
              for (int qd = 0; qd < 4; ++qd) hv[qd] = hn[qd];
            }
          }
          if (half == 0) {
            if (lane == 0) ptx::bulk_wait_read<L::kStagingBufs - 1>();  // this staging buffer's last store has read it
            __syncwarp();
          }
          // 32 bf16 = 4 x 16 B per row; SWIZZLE_64B: chunk ^= (row >> 1) & 3
#pragma unroll
          for (int j = 0; j < 2; ++j)
            *reinterpret_cast<uint4*>(st + lane * 64 + (((half * 2 + j) ^ ((lane >> 1) & 3)) << 4)) =
                make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]);
        }
        if (half == 1) {
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if constexpr (EPI == EPI_F32)
              ptx::tma_store_3d(&pr.map_out, st, col0, rbase, split);
            else
              ptx::tma_store_2d(&pr.map_out, st, col0, rbase + pr.out_row0);
            ptx::bulk_commit();
          }
          sbuf = (sbuf + 1) % L::kStagingBufs;
          gemm_stamp(etr, lt, (i >> 1) == 0 ? 5 : 9);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&tempty_bar[buf]);
        if constexpr (L::kAuxBufs > 0) ptx::mbar_arrive(&auxe_bar[lt % L::kAuxBufs]);
      }
      gemm_stamp(etr, lt, 6);
      if (nchain > 1 && ci + 1 < nchain && lane == 0) {
        // publish store completion for the next layer's producer: the previous tile's stores
        // (all but this tile's kUnits / 2 groups) without waiting, and everything at the layer's end
        if (tl + 1 == ntl) {
          ptx::bulk_wait<0>();
          __threadfence_block();
          stored_s[e] = lt + 1;
        } else {
          ptx::bulk_wait<kUnits / 2>();
          __threadfence_block();
          stored_s[e] = lt;
        }
      }
    }
    }
    if (lane == 0) ptx::bulk_wait<0>();
  } else if constexpr (CS) {
    // ---------------- column-sum warps (split-K weight gradient, A = dPre MN-major): while the
    // MMA consumes each A stage, sum its 64 K-rows for the tile's 128 M-columns (the layer's
    // bias gradient = column sums of dPre), then co-release the stage. CTAs with n0 == 0 write
    // one fp32 row per (split, m-tile): colsum[split * M + m].
    const int c = (warp - 2 - kEpiWarps) * 32 + lane;  // 0..127
    const int box = c >> 6, cc = c & 63;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntile_total; tile += gridDim.x) {
      int prob, split, m0, n0, kb0, nkb;
      decode(tile, prob, split, m0, n0, kb0, nkb);
      const GemmProblem& pr = P.prob[prob];
      const bool on = pr.colsum != nullptr && n0 == 0;
      float s = 0.f;
      for (int i = 0; i < nkb; ++i, ++it) {
        const int st = it % S;
        ptx::mbar_wait(&full_bar[st], (it / S) & 1);
        if (on) {
          const uint8_t* sa = smem + st * L::kStage + box * 8192 + (cc & 7) * 2;
#pragma unroll 8
          for (int r = 0; r < kGemmBlockK; ++r) {
            const uint16_t v = *reinterpret_cast<const uint16_t*>(sa + r * 128 + ((((cc >> 3) ^ (r & 7))) << 4));
            s += __uint_as_float(uint32_t(v) << 16);
          }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty_bar[st]);
      }
      if (on && m0 + c < pr.M) pr.colsum[(long long)split * pr.M + m0 + c] = s;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem_base, L::kTmemCols);
}

}  // namespace gmi
