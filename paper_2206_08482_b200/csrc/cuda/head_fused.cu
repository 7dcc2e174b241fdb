// Fused PPO head step of one minibatch (K6 + the head parts of K4/K7): for each
// 128-row tile of the last hidden activations H_L of one net,
//   MMA1  head forward        mu | v  = H_L W_head^T           (N = 16 / 32, fp32 in TMEM)
//   loss  clipped surrogate / value loss per row -> G = dL/dmu | dL/dv (bf16, smem operand)
//   MMA2  head input grad     acc    = G W_head                (N = hp)
//   epi   dPre_{L-1} = acc * elu'(H_L) (H_L read from the smem tile) -> bf16 -> TMA store
//   MMA3  head weight grad    dW^T  += H_L^T G                 (accumulated in TMEM over all
//         tiles of the CTA; one fp32 slab per CTA)
// so the head forward, the loss and the head input- and weight-gradient GEMMs become one
// launch, and mu / v / G never touch HBM. Column group 0 (4 warps) runs the per-row loss while
// groups 1-3 run the elu' epilogue of the previous tile.
//
// CTAs [0, npol) serve the policy net (0), the rest the value net (1); CTA c of a net takes that
// net's tiles c, c + ctas, ...
// Warp 0: TMA (head weights once, H tiles), warp 1: tcgen05.mma issuer, warps 2..17:
// epilogue (warps with column group 0 also run the per-row loss). Per-CTA partial outputs
// (weight-grad slab, bias-grad row, head-bias / log-std grads and loss statistics) are summed
// in a fixed order by the gradient-assembly kernel, so results are deterministic.
// Numerics follow head_loss_kernel / oracle/ppo_oracle.c.
#include <cuda.h>
#include <algorithm>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../host/errors.hpp"
#include "gemm.cuh"
#include "head_fused.cuh"
#include "head_loss.cuh"
#include "launch.cuh"
#include "ppo_common.cuh"

namespace gmi::ppo {

namespace {

constexpr int kRows = 128;
constexpr int kEpiWarps = 16;
constexpr int kThreads = 64 + 32 * kEpiWarps + 32;  // TMA, MMA, epilogue warps, MMA3 warp (last)
constexpr uint32_t kChunk = kRows * 128;  // [128 rows][64 bf16], SW128
constexpr uint32_t kOffH = 0;              // 2 x H_L tile (double-buffered), 4 K-chunks each
constexpr uint32_t kOffG = 8 * kChunk;     // 2 x G tile [128][64] bf16 (double-buffered, see MMA3)
constexpr uint32_t kOffWK = kOffG + 2 * kChunk;  // W_head K-major, per K-chunk [32 rows][128 B]
constexpr uint32_t kOffWM = kOffWK + 4 * 4096;  // W_head MN-major, [32 K-rows][64 cols] boxes
constexpr int kElu = 12;  // warps on the elu' epilogue (column groups 1..3); group 0 runs the loss
constexpr uint32_t kOffStg = kOffWM + 4 * 4096;  // epilogue staging, 2 KB per elu' warp
constexpr uint32_t kOffRed = kOffStg + kElu * 2048;  // 4 x 256 fp32
constexpr uint32_t kOffBar = kOffRed + 4 * 256 * 4;
constexpr uint32_t kSmem = kOffBar + 768 + 1024;  // barriers + per-action constants (128 floats)
static_assert(kSmem <= 232448, "shared memory budget");
constexpr uint32_t kTmemAcc1 = 0, kTmemAcc3 = 64, kTmemAcc2 = 256;  // acc1: 2 x 32 columns

// Development trace (`make TRACE=1`): globaltimer stamps of CTA 0, tiles 0..3, into a buffer
// set with head_fused_set_trace (tools: get("head_trace")).
__device__ unsigned long long* g_head_trace = nullptr;
__device__ __forceinline__ void hstamp(bool on, int it, int k) {
#ifdef GMI_TRACE
  if (on && g_head_trace && blockIdx.x == 0 && it < 4) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_head_trace[it * 16 + k] = t;
  }
#else
  (void)on, (void)it, (void)k;
#endif
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory"); }
// the four loss warps (column group 0: warps 2..5)
__device__ __forceinline__ void loss_bar() { asm volatile("bar.sync 2, 128;" ::: "memory"); }

template <int MAXA>
__global__ void __launch_bounds__(kThreads, 1) head_fused_kernel(const __grid_constant__ HeadFusedArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::align_smem_1024(smem_raw);
  uint8_t* sH = smem + kOffH;
  uint8_t* sG = smem + kOffG;
  uint8_t* sWK = smem + kOffWK;
  uint8_t* sWM = smem + kOffWM;
  float* red = reinterpret_cast<float*>(smem + kOffRed);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* wbar = bars;
  uint64_t* hfull = bars + 1;  // [2]
  uint64_t* hfree = bars + 3;  // [2]
  // G(t) published: one barrier per G buffer (t & 1), so a barrier's phase advances once per two
  // tiles and a waiter can never miss a phase (the loss of tile t+2 needs MMA3(t) first)
  uint64_t* g_ready2[2] = {bars + 5, bars + 12};
  uint64_t* acc2_full = bars + 6;
  uint64_t* acc2_free = bars + 7;
  uint64_t* fin = bars + 8;
  uint64_t* acc1_full = bars + 9;  // [2]: double-buffered head output
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int net = int(blockIdx.x) < a.npol ? 0 : 1;
  const int cta = net ? int(blockIdx.x) - a.npol : int(blockIdx.x);
  const int ctas = net ? int(gridDim.x) - a.npol : a.npol;
  const HeadNet& hn = a.net[net];
  const int hp = a.hp, nk = (hp + 63) / 64, NH = hn.nh, nout = hn.n_out;
  const int mtiles = (a.Bm + kRows - 1) / kRows;

  if (threadIdx.x == 0) {
    ptx::mbar_init(wbar, 1);
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&hfull[b], 1);
      ptx::mbar_init(&hfree[b], kElu + 1);  // elu' epilogue reads + MMA3 commit
    }
    ptx::mbar_init(&acc1_full[0], 1);
    ptx::mbar_init(&acc1_full[1], 1);
    ptx::mbar_init(g_ready2[0], 1);  // one arrival per tile, after all four loss warps (see below)
    ptx::mbar_init(g_ready2[1], 1);
    ptx::mbar_init(acc2_full, 1);
    ptx::mbar_init(acc2_free, kElu);
    ptx::mbar_init(fin, 1);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&hn.map_h);
    ptx::tma_prefetch_desc(&hn.map_wk);
    ptx::tma_prefetch_desc(&hn.map_wm);
    ptx::tma_prefetch_desc(&hn.map_d);
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  // G tile: columns >= n_out must be zero (they are the K padding of MMA2 / N padding of MMA3)
  for (int i = threadIdx.x; i < int(2 * kChunk / 16); i += blockDim.x)
    reinterpret_cast<uint4*>(sG)[i] = make_uint4(0u, 0u, 0u, 0u);
  ptx::fence_proxy_async_smem();
  pdl_trigger();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(wbar, uint32_t(nk) * (uint32_t(NH) * 128u + 4096u));
      for (int kc = 0; kc < nk; ++kc) {
        ptx::tma_load_2d(sWK + kc * 4096, &hn.map_wk, wbar, kc * 64, 0);
        ptx::tma_load_2d(sWM + kc * 4096, &hn.map_wm, wbar, kc * 64, 0);
      }
      int it = 0;
      for (int j = cta; j < mtiles; j += ctas, ++it) {
        const int b = it & 1;
        if (it >= 2) ptx::mbar_wait_sleep(&hfree[b], ((it >> 1) - 1) & 1);
        ptx::mbar_arrive_expect_tx(&hfull[b], uint32_t(nk) * kChunk);
        for (int kc = 0; kc < nk; ++kc)
          ptx::tma_load_2d(sH + (b * 4 + kc) * kChunk, &hn.map_h, &hfull[b], kc * 64, j * kRows);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      ptx::mbar_wait_sleep(wbar, 0);
      const uint32_t idesc1 = ptx::umma_idesc_bf16(kRows, uint32_t(NH), 0, 0);
      const uint32_t idesc2 = ptx::umma_idesc_bf16(kRows, uint32_t((hp + 15) / 16 * 16), 0, 1);
      const uint32_t g0 = ptx::smem_u32(sG);
      const uint32_t wk0 = ptx::smem_u32(sWK), wm0 = ptx::smem_u32(sWM);
      // MMA1 of tile t+1 overlaps tile t's loss (double-buffered head output, acc1_full[t & 1])
      auto mma1 = [&](int t) {
        const int b = t & 1;
        const uint32_t h0 = ptx::smem_u32(sH + b * 4 * kChunk);
        hstamp(true, t, 0);
        ptx::mbar_wait(&hfull[b], (t >> 1) & 1);
        hstamp(true, t, 1);
        ptx::tc_fence_after();
        // MMA1: [128 x NH] = H . W_head^T (K = hp)
        for (int kc = 0; kc < nk; ++kc) {
          const int ks = min(4, (hp - kc * 64 + 15) / 16);
          for (int k = 0; k < ks; ++k)
            ptx::mma_bf16(tmem + kTmemAcc1 + b * 32, ptx::umma_desc_sw128(h0 + kc * kChunk + k * 32, 16, 1024),
                          ptx::umma_desc_sw128(wk0 + kc * 4096 + k * 32, 16, 1024), idesc1,
                          (kc > 0 || k > 0) ? 1u : 0u);
        }
        ptx::mma_commit(&acc1_full[b]);
        hstamp(true, t, 2);
      };
      const int ntiles = cta < mtiles ? (mtiles - cta + ctas - 1) / ctas : 0;
      int next1 = 0;  // first tile whose MMA1 is not issued yet
      for (int it = 0; it < ntiles; ++it) {
        // MMA2(it) as soon as its G is ready and acc2 is drained; meanwhile MMA1 of the next
        // tile is issued the moment its H tile lands (acc1 is double-buffered: at most one ahead)
        while (true) {
          if (next1 < ntiles && next1 <= it + 1 && ptx::mbar_test(&hfull[next1 & 1], (next1 >> 1) & 1)) {
            mma1(next1);
            ++next1;
          }
          if (next1 > it && ptx::mbar_test(g_ready2[it & 1], (it >> 1) & 1) && (it == 0 || ptx::mbar_test(acc2_free, (it - 1) & 1)))
            break;
        }
        const uint32_t gt = g0 + (it & 1) * kChunk;
        hstamp(true, it, 3);
        ptx::tc_fence_after();
        // MMA2: [128 x hp] = G . W_head (K = NH; W_head read MN-major)
        for (int k = 0; k < NH / 16; ++k)
          ptx::mma_bf16(tmem + kTmemAcc2, ptx::umma_desc_sw128(gt + k * 32, 16, 1024),
                        ptx::umma_desc_sw128(wm0 + k * 2048, 4096, 1024), idesc2, k > 0 ? 1u : 0u);
        ptx::mma_commit(acc2_full);
        hstamp(true, it, 4);
      }
    }
  } else if (warp == 2 + kEpiWarps) {
    // ------------------------------------------------ MMA3 issuer: the head weight gradient
    // dW_head^T[hp x NH] += H^T . G (K = tile rows; both operands MN-major views), accumulated in
    // TMEM over the CTA's tiles. A thread of its own: its 16 small-N MMAs take ~1.3 us to issue
    // and would otherwise delay the next tile's MMA1 / MMA2. G is double-buffered: the loss of
    // tile t+2 only starts after MMA1(t+2), whose H tile could load only after MMA3(t) freed it.
    if (lane == 0) {
      ptx::mbar_wait_sleep(wbar, 0);
      const uint32_t idesc3 = ptx::umma_idesc_bf16(kRows, uint32_t(NH), 1, 1);
      const uint32_t g0 = ptx::smem_u32(sG);
      int it = 0;
      for (int j = cta; j < mtiles; j += ctas, ++it) {
        const uint32_t h0 = ptx::smem_u32(sH + (it & 1) * 4 * kChunk);
        const uint32_t gt = g0 + (it & 1) * kChunk;
        ptx::mbar_wait_sleep(g_ready2[it & 1], (it >> 1) & 1);  // G(t) written; H(t) landed before MMA1(t)
        ptx::tc_fence_after();
        for (int half = 0; half * 128 < hp; ++half)
          for (int k = 0; k < kRows / 16; ++k)
            ptx::mma_bf16(tmem + kTmemAcc3 + half * 32,
                          ptx::umma_desc_sw128(h0 + 2 * half * kChunk + k * 2048, kChunk, 1024),
                          ptx::umma_desc_sw128(gt + k * 2048, 8192, 1024), idesc3, (it > 0 || k > 0) ? 1u : 0u);
        ptx::mma_commit(&hfree[it & 1]);
      }
      ptx::mma_commit(fin);
    }
  } else {
    // ------------------------------------------------ epilogue warps
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const float invB = 1.0f / float(a.Bm);
    uint8_t* stg = smem + kOffStg + (h > 0 ? warp - 6 : 0) * 2048;  // elu' warps only
    // per-action constants of the loss, once per CTA: log_std, exp(log_std), head bias
    float* cst = reinterpret_cast<float*>(smem + kOffBar + 128);
    float* lacc = red + q * 128;  // this lane quarter's per-action sums [0, 64) and statistics [64, 68)
    if (threadIdx.x - 64 < a.A) {
      const float ls = a.log_std[threadIdx.x - 64];
      cst[threadIdx.x - 64] = ls;
      cst[32 + threadIdx.x - 64] = expf(ls);
      cst[96 + threadIdx.x - 64] = 1.0f / expf(ls);
    }
    if (threadIdx.x - 64 < nout) cst[64 + threadIdx.x - 64] = hn.bias[threadIdx.x - 64];
    if (h == 0 && lane == 0)
      for (int i = 0; i < 128; ++i) lacc[i] = 0.f;
    epi_bar();
    float st[4] = {0.f, 0.f, 0.f, 0.f};
    float sg[kLossRegAcc<MAXA> ? MAXA : 1], sl[kLossRegAcc<MAXA> ? MAXA : 1];  // running per-action sums (A <= 8)
#pragma unroll
    for (int i = 0; i < (kLossRegAcc<MAXA> ? MAXA : 1); ++i) sg[i] = sl[i] = 0.f;
    int it = 0;
    for (int j = cta; j < mtiles; j += ctas, ++it) {
      const int grow = j * kRows + row;
      const bool valid = grow < a.Bm;
      if (h == 0) {
        // ---- per-row loss (thread = row): TMEM lane quarter q. The row's stored action, old
        // log-prob, advantage and return are fetched before the accumulator wait so their
        // latency overlaps the head MMA.
        const long long rr = a.row0 + grow;
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
        ptx::mbar_wait_sleep(&acc1_full[it & 1], (it >> 1) & 1);
        hstamp(warp == 2 && lane == 0, it, 5);
        ptx::tc_fence_after();
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem + kTmemAcc1 + (it & 1) * 32 + (static_cast<uint32_t>(q * 32) << 16), r);
        ptx::tmem_ld_wait();
        head_row_loss<MAXA>(net, r, cst, nout, NH, valid, a.act + rr * nout, act_r, oldlp, adv, ret, a.clip,
                            a.vf_coef, a.ent_coef, invB, sG + (it & 1) * kChunk + row * 128, row, lacc, st, sg, sl);
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        // All four loss warps finish tile `it` before G(it) is published. With one arrival per
        // warp on a count-4 barrier, a warp that ran ahead could arrive for tile it+1 (its
        // accumulator is double-buffered and MMA1(it+1) may already be done) and complete tile
        // it's phase while a slower warp's G rows were still unwritten (MMA2 / MMA3 then read
        // them stale: nondeterministic gradients, ~1 run in 10 at the bench shape).
        loss_bar();
        if (warp == 2 && lane == 0) ptx::mbar_arrive(g_ready2[it & 1]);
        hstamp(warp == 2 && lane == 0, it, 6);
      }

      // ---- dPre_{L-1} = (G W_head) * elu'(H_L) on column groups 1..3 (chunks c = h-1, h+2, h+5),
      // so group 0 can already run the next tile's loss
      if (h == 0) continue;
      ptx::mbar_wait_sleep(acc2_full, it & 1);
      hstamp(warp == 6 && lane == 0, it, 7);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int pass = 0; pass < 3; ++pass) {
        const int c = (h - 1) + 3 * pass;
        if (c * 32 >= hp) break;
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem + kTmemAcc2 + (static_cast<uint32_t>(q * 32) << 16) + c * 32, r);
        // H_L row `row`, columns 32c..32c+31: 4 x 16 B from the swizzled operand tile
        const uint8_t* hrow = sH + ((it & 1) * 4 + (c >> 1)) * kChunk + row * 128;
        uint4 hv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          hv[u] = *reinterpret_cast<const uint4*>(hrow + ((((c & 1) * 4 + u) ^ (row & 7)) << 4));
        ptx::tmem_ld_wait();
        uint32_t packed[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t hw[4] = {hv[u].x, hv[u].y, hv[u].z, hv[u].w};
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const int jj = u * 8 + x * 2;
            const float2 d = dact2(make_float2(__uint_as_float(r[jj]), __uint_as_float(r[jj + 1])), hw[x]);
            packed[jj / 2] = pack_bf16(d.x, d.y);
          }
        }
        if (lane == 0) ptx::bulk_wait_read<0>();  // the staging buffer's previous store has read it
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 4; ++u)
          *reinterpret_cast<uint4*>(stg + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4)) =
              make_uint4(packed[4 * u], packed[4 * u + 1], packed[4 * u + 2], packed[4 * u + 3]);
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          ptx::tma_store_2d(&hn.map_d, stg, c * 32, j * kRows + q * 32);
          ptx::bulk_commit();
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(acc2_free);
        hstamp(warp == 6, it, 8);
        ptx::mbar_arrive(&hfree[it & 1]);
      }
    }

    // ---- per-CTA outputs
    // (b) head weight gradient slab: TMEM rows = hp index, columns = head outputs
    ptx::mbar_wait_sleep(fin, 0);
    ptx::tc_fence_after();
    if (h < 2 && h * 128 < hp) {
      uint32_t r[32];
      ptx::tmem_ld_32x32b_x32(tmem + kTmemAcc3 + h * 32 + (static_cast<uint32_t>(q * 32) << 16), r);
      ptx::tmem_ld_wait();
      const int k = h * 128 + row;
      if (k < hp)
        for (int o = 0; o < nout; ++o)
          hn.dw_slab[((long long)cta * nout + o) * hp + k] = (it > 0) ? __uint_as_float(r[o]) : 0.f;
    }
    // (c) head-bias / log-std gradients and loss statistics: per-quarter records in `red`
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
            src < 0 ? 0.f : ((red[src] + red[128 + src]) + red[256 + src]) + red[384 + src];
      }
    if (lane == 0) ptx::bulk_wait<0>();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

}  // namespace

void head_fused_set_trace(unsigned long long* buf) {
  GMI_CUDA_CHECK(cudaMemcpyToSymbol(g_head_trace, &buf, sizeof(buf)));
}

bool head_fusable(int hp, int A) { return hp <= 256 && A <= 31 && A >= 1; }

int head_fused_grid(int Bm, int sms) {
  const int tiles = (Bm + kRows - 1) / kRows;
  const int per_net = std::max(1, std::min(tiles, sms / 2));
  return 2 * per_net;
}

int head_fused_npol(int grid, int A) {
  if (const char* e = std::getenv("GMI_HEAD_NPOL")) {  // measurement override
    const int n = std::atoi(e);
    if (n > 0 && n < grid) return n;
  }
  // CTAs in proportion to the per-tile cost: a policy tile (A log-probs, ratio, clip, per-action
  // gradients) costs r value tiles, r measured on B200 from the policy-CTA sweeps of
  // profiles/r2/SUMMARY.md (AT, A = 8: best split 80 / 68, r ~ 1.2; HM, A = 21: 110-120 / 38-28,
  // r ~ 3), interpolated linearly in A
  const double r = std::max(1.0, 1.2 + (3.0 - 1.2) / 13.0 * (A - 8));
  const int n = int(grid * r / (1.0 + r) + 0.5);
  return std::max(1, std::min(grid - 1, n));
}

void launch_head_fused(const HeadFusedArgs& a, int grid, cudaStream_t s) {
  if (a.npol < 1 || a.npol >= grid) invalid("head kernel: policy CTA count out of range");
  auto go = [&](auto kern) {
    static bool configured[4] = {};
    (void)configured;
    GMI_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    launch_pdl(kern, dim3(grid), dim3(kThreads), kSmem, s, a);
  };
  if (a.A <= 8)
    go(head_fused_kernel<8>);
  else if (a.A <= 16)
    go(head_fused_kernel<16>);
  else if (a.A <= 24)
    go(head_fused_kernel<24>);
  else
    go(head_fused_kernel<31>);
}

}  // namespace gmi::ppo
