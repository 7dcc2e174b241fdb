// Fused rollout, cluster variant: C CTAs (C = hidden width / 64) share one 128-env tile.
//
// Each CTA of the cluster owns a 64-column slice of every hidden layer: it keeps that slice
// of the weights resident in shared memory for the whole rollout (no per-step weight
// streaming), computes its 128 x 64 slice of the layer output (tcgen05.mma N = 64), and
// all-gathers the slices through distributed shared memory: the slice is exactly one 64-column
// K-chunk of the next layer's SW128 operand tile, so each CTA writes it locally and pushes it to
// the C-1 peers with cp.async.bulk shared::cta -> shared::cluster, completing on the peer's
// operand-tile mbarrier. The policy head (N = 16) is computed redundantly by every CTA; CTA r
// then steps its 32 envs (16 threads per env: actions, dynamics on register-resident state,
// reward, reset) and all-gathers the next observation rows the same way.
//
// Why: the single-CTA kernel (rollout.cu) serialises MMA -> 32K-element epilogue -> env step on
// one SM per 128 envs and streams ~290 KB of weights per step; splitting N over C SMs cuts the
// per-step chain ~C-fold and keeps weights on chip.
//
// Synchronisation (no cluster barrier inside the loop): operand tile b = layer parity has one
// mbarrier whose phase completes when the local slice is written (one local arrive.expect_tx of
// the peers' bytes) and the C-1 peer slices have landed (complete_tx). A peer can only push
// layer l's slice after its own MMA(l), which needed this CTA's layer l-1 slice, which this CTA
// produced after its own MMA(l-1) finished reading the tile being overwritten -- so neither
// WAR nor phase-overrun hazards exist (requires an odd number of hidden layers so the head
// never reads the observation tile). Numerics are identical to rollout.cu.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

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
constexpr uint32_t kChunk = kRows * 128;        // 64-column K-chunk of a 128-row tile (16 KB)
constexpr uint32_t kAct = 4 * kChunk;           // 128 x 256 bf16
constexpr uint32_t kWChunk = 64 * 128;          // [64 rows][64 K] bf16 slice chunk (8 KB)
constexpr uint32_t kHChunk = 16 * 128;          // [16 rows][64 K] head chunk (2 KB)
constexpr uint32_t kOffW = 2 * kAct;            // resident weight slices
constexpr uint32_t kWBytes = kWChunk + 2 * 4 * kWChunk;  // layer 0 (1 chunk) + 2 hidden (4 chunks)
constexpr uint32_t kOffHead = kOffW + kWBytes;
constexpr uint32_t kOffMu = kOffHead + 4 * kHChunk;     // mu / tanh(u) staging [32][17] x 2
constexpr int kMuLd = 17;
constexpr uint32_t kOffBar = kOffMu + 2 * 32 * kMuLd * 4 + 64;
constexpr uint32_t kSmem = kOffBar + 256 + 1024;
constexpr int kMaxL = 3;

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory"); }

__device__ __forceinline__ void trace_at(const RolloutArgs& a, int idx) {  // development aid
  if (a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[idx] = t;
  }
}

__device__ __forceinline__ uint32_t sw128(int row, int col_bf16) {
  const int u = (col_bf16 & 63) >> 3;
  return uint32_t(row * 128 + ((u ^ (row & 7)) << 4) + (col_bf16 & 7) * 2);
}

template <int C>
__global__ void __launch_bounds__(kThreads, 1) rollout_cluster_kernel(const __grid_constant__ RolloutArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::align_smem_1024(smem_raw);
  uint8_t* act[2] = {smem, smem + kAct};
  uint8_t* wsl = smem + kOffW;
  uint8_t* whd = smem + kOffHead;
  float* mu_s = reinterpret_cast<float*>(smem + kOffMu);
  float* u_s = mu_s + 32 * kMuLd;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* wbar = bars;
  uint64_t* act_full = bars + 1;  // [2]
  uint64_t* acc_full = bars + 3;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
  float* ls_s = reinterpret_cast<float*>(bars + 8);  // [16] log_std, [16] exp(log_std)
  float* sig_s = ls_s + 16;
  // per K-chunk arrival of a hidden layer's all-gathered output ([buffer][chunk = producing CTA]):
  // the next layer's MMAs on chunk kc start as soon as that slice is here, in the fixed kc order
  uint64_t* chunk_full = bars + 24;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = a.L, T = a.T;
  const int rank = int(ptx::cluster_rank());
  const int m0 = (blockIdx.x / C) * kRows;  // the cluster's 128-env tile
  // weight-slice chunk offsets: layer 0 = 1 chunk (S_p <= 64), hidden layers C chunks
  auto wl = [&](int l) { return wsl + (l == 0 ? 0u : kWChunk + uint32_t(l - 1) * C * kWChunk); };

  if (threadIdx.x == 0) {
    ptx::mbar_init(wbar, 1);
    ptx::mbar_init(&act_full[0], 1);
    ptx::mbar_init(&act_full[1], 1);
    for (int i = 0; i < 2 * C; ++i) ptx::mbar_init(&chunk_full[i], 1);
    ptx::mbar_init(acc_full, 1);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&a.map_obs);
    for (int l = 0; l <= L; ++l) ptx::tma_prefetch_desc(&a.map_w[l]);
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 256);
  pdl_trigger();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // every CTA's barriers exist before any peer pushes into them
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer: resident weights, first obs
    if (lane == 0) {
      uint32_t bytes = kWChunk + uint32_t(L - 1) * C * kWChunk + uint32_t(C) * kHChunk;
      ptx::mbar_arrive_expect_tx(wbar, bytes);
      ptx::tma_load_2d(wl(0), &a.map_w[0], wbar, 0, 64 * rank);
      for (int l = 1; l < L; ++l)
        for (int kc = 0; kc < C; ++kc) ptx::tma_load_2d(wl(l) + kc * kWChunk, &a.map_w[l], wbar, kc * 64, 64 * rank);
      for (int kc = 0; kc < C; ++kc) ptx::tma_load_2d(whd + kc * kHChunk, &a.map_w[L], wbar, kc * 64, 0);
      ptx::mbar_arrive_expect_tx(&act_full[0], kChunk);
      ptx::tma_load_2d(act[0], &a.map_obs, &act_full[0], 0, m0);
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      ptx::mbar_wait(wbar, 0);
      int obs_ph = 0, cph[2] = {0, 0}, acc_ph = 0;
      const uint32_t idesc_h = ptx::umma_idesc_bf16(kRows, 64, 0, 0);
      const uint32_t idesc_o = ptx::umma_idesc_bf16(kRows, 16, 0, 0);
      for (int t = 0; t < T; ++t)
        for (int l = 0; l <= L; ++l) {
          const int b = l & 1;
          if (l == 0) ptx::mbar_wait(&act_full[0], (obs_ph++) & 1);  // observation rows of all 4 CTAs
          ptx::tc_fence_after();
          const bool head = l == L;
          const uint32_t acc = tmem + (head ? 128u : uint32_t(acc_ph++ & 1) * 64u);
          const uint32_t in = ptx::smem_u32(act[b]);
          const uint32_t wb = ptx::smem_u32(head ? whd : wl(l));
          const uint32_t cstride = head ? kHChunk : kWChunk;
          const int K = a.in_p[l];
          const int nk = (K + 63) / 64;
          for (int kc = 0; kc < nk; ++kc) {
            if (l > 0) {  // slice kc of the previous layer (local or pushed by CTA kc)
              ptx::mbar_wait(&chunk_full[b * C + kc], cph[b] & 1);
              ptx::tc_fence_after();
            }
            const int ks = min(4, (K - kc * 64 + 15) / 16);
            for (int k = 0; k < ks; ++k)
              ptx::mma_bf16(acc, ptx::umma_desc_sw128(in + kc * kChunk + k * 32, 16, 1024),
                            ptx::umma_desc_sw128(wb + kc * cstride + k * 32, 16, 1024), head ? idesc_o : idesc_h,
                            (kc > 0 || k > 0) ? 1u : 0u);
          }
          if (l > 0) ++cph[b];
          ptx::mma_commit(acc_full);
        }
    }
  } else {
    // ------------------------------------------------ epilogue + env threads
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const int tid = threadIdx.x - 64;
    const int el = tid >> 4, sub = tid & 15;  // 32 envs of this CTA, 16 threads each
    const int env = m0 + rank * 32 + el;
    const bool valid = env < a.N;
    const int gid = a.env0 + env;
    const int A = a.A, S = a.S, S_p = a.S_p;
    const int base = lane & ~15;  // first lane of this env's 16-lane group
    const int blk = sub;          // the thread's 4-dim state block
    const bool owns = valid && blk * 4 < S;
    float xs[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = blk * 4 + j;
      xs[j] = owns && i < S ? a.x[(long long)env * S + i] : 0.f;
    }
    const float rA = 1.0f / float(A);  // action index of a state dim: i % A via an fp32 reciprocal
    int st = 0, len = 1, cnt = 0;
    if (valid) {
      st = a.ep_step[env];
      len = a.ep_len[env];
      cnt = a.ep_count[env];
    }
    if (tid < A) {
      const float ls = a.log_std[tid];
      ls_s[tid] = ls;
      sig_s[tid] = expf(ls);
    }
    const uint32_t it0 = uint32_t(a.ctl->iteration) * uint32_t(T);
    const uint32_t act_base[2] = {ptx::smem_u32(act[0]), ptx::smem_u32(act[1])};
    int accph = 0, acc_ph = 0;
    for (int t = 0; t < T; ++t) {
      for (int l = 0; l < L; ++l) {
        const uint32_t acc = tmem + uint32_t(acc_ph++ & 1) * 64u;
        ptx::mbar_wait_sleep(acc_full, (accph++) & 1);
        ptx::tc_fence_after();
        trace_at(a, t * 16 + 2 * l);
        uint32_t r[16];
        ptx::tmem_ld_32x32b_x16(acc + (static_cast<uint32_t>(q * 32) << 16) + h * 16, r);
        const float4* b4 = reinterpret_cast<const float4*>(a.bias[l] + rank * 64 + h * 16);
        float4 bb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) bb[j] = __ldg(b4 + j);
        ptx::tmem_ld_wait();
        uint32_t packed[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 y0 = bias_elu2(make_float2(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1])),
                                      make_float2(bb[j].x, bb[j].y));
          const float2 y1 = bias_elu2(make_float2(__uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])),
                                      make_float2(bb[j].z, bb[j].w));
          packed[2 * j] = pack_bf16(y0.x, y0.y);
          packed[2 * j + 1] = pack_bf16(y1.x, y1.y);
        }
        const int nb = (l + 1) & 1;
        uint8_t* chunk = act[nb] + rank * kChunk + row * 128;
#pragma unroll
        for (int u = 0; u < 2; ++u)
          *reinterpret_cast<uint4*>(chunk + (((2 * h + u) ^ (row & 7)) << 4)) =
              make_uint4(packed[4 * u], packed[4 * u + 1], packed[4 * u + 2], packed[4 * u + 3]);
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        epi_bar();
        trace_at(a, t * 16 + 2 * l + 1);
        if (tid == 0) {  // push the slice (one 16 KB K-chunk) to the peers' chunk `rank`, arm our
          // remote chunks and mark our own chunk ready
          const uint32_t src = act_base[nb] + rank * kChunk;
          const uint32_t bar = ptx::smem_u32(&chunk_full[nb * C + rank]);
#pragma unroll
          for (int p = 1; p < C; ++p) {
            const uint32_t peer = uint32_t((rank + p) % C);
            ptx::bulk_s2s(ptx::mapa(src, peer), src, kChunk, ptx::mapa(bar, peer));
          }
#pragma unroll
          for (int kc = 0; kc < C; ++kc) {
            if (kc == rank)
              ptx::mbar_arrive(&chunk_full[nb * C + kc]);
            else
              ptx::mbar_arrive_expect_tx(&chunk_full[nb * C + kc], kChunk);
          }
        }
      }

      // ---- head: mu for this CTA's 32 envs (TMEM lanes 32 rank ..)
      ptx::mbar_wait_sleep(acc_full, (accph++) & 1);
      ptx::tc_fence_after();
      trace_at(a, t * 16 + 10);
      if (q == rank && h == 0) {
        uint32_t r[16];
        ptx::tmem_ld_32x32b_x16(tmem + 128u + (static_cast<uint32_t>(q * 32) << 16), r);
        ptx::tmem_ld_wait();
        for (int i = 0; i < A; ++i) mu_s[lane * kMuLd + i] = __uint_as_float(r[i]) + a.bias[L][i];
      }
      ptx::tc_fence_before();
      epi_bar();

      // ---- actions: item w = (Philox block w/2, Box-Muller pair w%2); thread `sub` takes item sub
      const uint32_t step = it0 + uint32_t(t);
      float lp_part = 0.f, usq_part = 0.f;
      if (valid && sub < 2 * ((A + 3) / 4)) {
        const int pb = sub >> 1, p = sub & 1;
        uint32_t rr[4];
        rng::draw(a.seed, uint32_t(gid), step, uint32_t(pb), rng::kNoise, rr);
        const uint32_t r0 = p ? rr[2] : rr[0], r1 = p ? rr[3] : rr[1];
        const float rad = sqrtf(-2.0f * logf(rng::u01_open0(r0)));
        const float th = kTwoPi * rng::u01(r1);
        float sn, cs;
        sincosf(th, &sn, &cs);
        const float nrm[2] = {rad * cs, rad * sn};
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int ai = pb * 4 + 2 * p + j;
          if (ai < A) {
            const float mu = mu_s[el * kMuLd + ai];
            const float ls = ls_s[ai], sig = sig_s[ai];
            const float act_v = mu + sig * nrm[j];
            const float z = (act_v - mu) / sig;
            lp_part += -0.5f * z * z - ls - kLog2PiHalf;
            const float u = fminf(fmaxf(act_v, -1.f), 1.f);
            usq_part += u * u;
            u_s[el * kMuLd + ai] = tanhf(u);
            a.act[((long long)t * a.N + env) * A + ai] = act_v;
          }
        }
      }
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) {
        lp_part += __shfl_xor_sync(0xffffffffu, lp_part, o);
        usq_part += __shfl_xor_sync(0xffffffffu, usq_part, o);
      }
      __syncwarp();
      trace_at(a, t * 16 + 11);

      // ---- dynamics (thread = one 4-dim block; right neighbour of dim 4k+3 = first dim of
      // block k+1 held by lane sub+1, or dim 0 past the last state dim)
      const float x0 = __shfl_sync(0xffffffffu, xs[0], base);
      const float nx = __shfl_sync(0xffffffffu, xs[0], base + ((sub + 1) & 15));
      float xn[4] = {0.f, 0.f, 0.f, 0.f};
      float xsq_part = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = blk * 4 + j;
        if (owns && i < S) {
          const float nbv = i + 1 >= S ? x0 : j < 3 ? xs[j + 1] : nx;
          const float drive = u_s[el * kMuLd + (i - A * fdiv(i, A, rA))];
          const float inner = __fadd_rn(__fsub_rn(drive, __fmul_rn(kDamp, xs[j])), __fmul_rn(kCouple, env_sin(nbv)));
          xn[j] = __fadd_rn(xs[j], __fmul_rn(kDt, inner));
          xsq_part = __fadd_rn(xsq_part, __fmul_rn(xn[j], xn[j]));
        }
      }
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) xsq_part += __shfl_xor_sync(0xffffffffu, xsq_part, o);
      const float xn0 = __shfl_sync(0xffffffffu, xn[0], base);
      const bool done = st + 1 >= len;
      const int count = cnt + (done ? 1 : 0);
      if (valid && blk * 4 < S_p) {
        uint32_t rr[4] = {0u, 0u, 0u, 0u};
        if (done && blk * 4 < S) rng::draw(a.seed, uint32_t(gid), uint32_t(count), uint32_t(blk), rng::kReset, rr);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = blk * 4 + j;
          xs[j] = i >= S ? 0.f : done ? __fsub_rn(__fmul_rn(rng::u01(rr[j]), 0.2f), 0.1f) : xn[j];
        }
        const uint2 pk = make_uint2(pack_bf16(xs[0], xs[1]), pack_bf16(xs[2], xs[3]));
        *reinterpret_cast<uint2*>(a.X_roll + ((long long)(t + 1) * a.N + env) * S_p + blk * 4) = pk;
        if (t + 1 < T)  // next observation row into the layer-0 operand tile
          *reinterpret_cast<uint2*>(act[0] + sw128(rank * 32 + el, blk * 4)) = pk;
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
      trace_at(a, t * 16 + 12);
      if (t + 1 < T) {  // all-gather the 32 observation rows (4 KB of chunk 0) to the peers
        ptx::fence_proxy_async_smem();
        epi_bar();
        trace_at(a, t * 16 + 13);
        if (tid == 0) {  // push this CTA's 32 observation rows (4 KB of chunk 0) to the peers
          const uint32_t src = act_base[0] + rank * 32 * 128;
          const uint32_t bar = ptx::smem_u32(&act_full[0]);
#pragma unroll
          for (int p = 1; p < C; ++p) {
            const uint32_t peer = uint32_t((rank + p) % C);
            ptx::bulk_s2s(ptx::mapa(src, peer), src, 32 * 128, ptx::mapa(bar, peer));
          }
          ptx::mbar_arrive_expect_tx(&act_full[0], uint32_t(C - 1) * 32 * 128);
        }
      }
    }
    if (valid) {
      if (sub == 0) {
        a.ep_step[env] = st;
        a.ep_count[env] = cnt;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = blk * 4 + j;
        if (owns && i < S) a.x[(long long)env * S + i] = xs[j];
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // no CTA leaves while a peer may still read from or push into it
  if (warp == 1) ptx::tmem_dealloc(tmem, 256);
}

template <int C>
void launch_c(const RolloutArgs& a, cudaStream_t s) {
  auto kern = rollout_cluster_kernel<C>;
  static bool configured = false;
  if (!configured) {
    GMI_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    GMI_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(((a.N + kRows - 1) / kRows) * C);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  GMI_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a));
}

}  // namespace

int rollout_cluster_size(int L, const int* widths_p, int S_p, int A, int N) {
  if (L < 1 || L > kMaxL || (L & 1) == 0 || S_p > 64 || A > 16 || A < 1 || N % kRows != 0) return 0;
  const int w = widths_p[1];
  for (int l = 1; l <= L; ++l)
    if (widths_p[l] != w) return 0;
  if (w != 256) return 0;  // 4 CTAs x 64-column slices; CTA r steps envs 32r..32r+31
  return 4;
}

void launch_rollout_cluster(const RolloutArgs& a, int C, cudaStream_t s) {
  if (C != 4) invalid("cluster rollout needs 4 CTAs per env tile");
  launch_c<4>(a, s);
}

}  // namespace gmi::ppo
