// Weight-gradient GEMM on SM pairs (tcgen05 cta_group::2) for the 256-wide hidden layers:
//
//   slab[split][m][n] = sum_{k in split} dPre[k][m] * H[k][n]      (M = N = 256, K = rows)
//   colsum[split][m]  = sum_{k in split} dPre[k][m]                 (the layer's bias gradient)
//
// The single-CTA kernel (gemm.cuh, M = 128 per CTA) was L2-to-SM bandwidth bound on this
// problem: each CTA received 48 KB per 64-row k-block (its 128 dPre columns + all 256 H
// columns, 46 B/clk/SM measured) for 2.1 MFLOP. Here the two CTAs of a cluster form one
// M = 256 tile: CTA r loads dPre columns [128 r, 128 r + 128) and H columns [128 r, 128 r + 128)
// (16 + 16 KB per k-block), and the leader issues tcgen05.mma.cta_group::2 (M = 256, N = 256),
// whose B operand is the union of both CTAs' H halves -- each SM now receives 32 KB per k-block
// for the same 2.1 MFLOP. Each CTA's TMEM holds its 128 output rows x 256 columns; its epilogue
// writes those rows of the split's fp32 slab, so the slab layout (and the fixed-order gradient
// assembly after it) is unchanged.
//
// Roles per CTA: warp 0 TMA producer (own halves, own full barrier); warp 1 lane 0 = MMA issuer
// in the leader / forwarder in the peer (waits its own full barrier, then arrives remotely on
// the leader's peer-full barrier, so the leader knows both halves landed); 8 epilogue warps
// (TMEM -> swizzled smem -> TMA store of the fp32 slab); 4 column-sum warps (sum of the CTA's
// dPre half over each stage's 64 rows). The leader's MMA commits multicast to both CTAs'
// empty / accumulator-full barriers; accumulator-empty arrivals of the peer are remote.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../host/errors.hpp"
#include "gemm_host.hpp"
#include "launch.cuh"
#include "ptx.cuh"

namespace gmi {

namespace {

constexpr int kPS = 6;                          // pipeline stages
constexpr uint32_t kHalf = 64 * 128 * 2;        // [64 K rows][128 cols] bf16 MN-major: 2 x [64][64] boxes
constexpr uint32_t kPStage = 2 * kHalf;         // dPre half + H half
constexpr int kPEpiWarps = 8;
constexpr uint32_t kPStaging = 4096;            // one 32 x 32 fp32 chunk per warp
constexpr uint32_t kPBarOff = kPS * kPStage + kPEpiWarps * kPStaging;
constexpr uint32_t kPSmem = kPBarOff + 256 + 1024;
constexpr int kPThreads = 64 + 32 * kPEpiWarps + 128;
constexpr uint32_t kIdesc = ptx::umma_idesc_bf16(256, 256, 1, 1);
static_assert(kPSmem <= 232448, "shared memory budget");

__device__ __forceinline__ void mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on `bar` (same smem offset) in both CTAs of the pair once the issued MMAs are done.
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          ptx::smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}

__device__ __forceinline__ void arrive_remote(uint64_t* bar, uint32_t rank) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   ptx::mapa(ptx::smem_u32(bar), rank))
               : "memory");
}

__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(ptx::smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPThreads, 1)
    gemm_pair_kernel(const __grid_constant__ GemmParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::align_smem_1024(smem_raw);
  uint8_t* staging = smem + kPS * kPStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPBarOff);
  uint64_t* empty = full + kPS;
  uint64_t* pfull = empty + kPS;   // leader: the peer's half of stage s landed
  uint64_t* tfull = pfull + kPS;   // [2]
  uint64_t* tempty = tfull + 2;    // [2] (leader: own + peer epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int ntile = P.num_problems * P.splits;
  const int nkb_total = (P.prob[0].K + kGemmBlockK - 1) / kGemmBlockK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPS; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1 + 4);  // leader's multicast MMA commit + 4 column-sum warps
      ptx::mbar_init(&pfull[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 2 * kPEpiWarps);
    }
    ptx::fence_mbar_init();
    for (int i = 0; i < P.num_problems; ++i) {
      ptx::tma_prefetch_desc(&P.prob[i].map_a);
      ptx::tma_prefetch_desc(&P.prob[i].map_b);
      ptx::tma_prefetch_desc(&P.prob[i].map_out);
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(tmem_slot)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  pdl_trigger();
  ptx::tc_fence_before();
  ptx::cluster_sync();  // barriers of both CTAs initialised before any remote arrive
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  auto decode = [&](int t, int& prob, int& split, int& kb0, int& nkb) {
    prob = t / P.splits;
    split = t - prob * P.splits;
    kb0 = split * P.prob[prob].kb_per_split;
    const int kb1 = min(nkb_total, kb0 + P.prob[prob].kb_per_split);
    nkb = kb1 > kb0 ? kb1 - kb0 : 0;
  };

  if (warp == 0) {
    // ---------------- TMA producer: this CTA's dPre and H halves
    if (lane == 0) {
      int it = 0;
      for (int t = cid; t < ntile; t += ncl) {
        int prob, split, kb0, nkb;
        decode(t, prob, split, kb0, nkb);
        const GemmProblem& pr = P.prob[prob];
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % kPS;
          if (it >= kPS) ptx::mbar_wait(&empty[s], ((it / kPS) - 1) & 1);
          uint8_t* sa = smem + s * kPStage;
          const int k0 = (kb0 + i) * kGemmBlockK;
          ptx::mbar_arrive_expect_tx(&full[s], kPStage);
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            ptx::tma_load_2d(sa + j * 8192, &pr.map_a, &full[s], int(rank) * 128 + 64 * j, k0 + pr.a_row0);
            ptx::tma_load_2d(sa + kHalf + j * 8192, &pr.map_b, &full[s], int(rank) * 128 + 64 * j, k0 + pr.b_row0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (leader): M = 256 (both CTAs' dPre halves), N = 256
      int it = 0, lt = 0;
      for (int t = cid; t < ntile; t += ncl, ++lt) {
        int prob, split, kb0, nkb;
        decode(t, prob, split, kb0, nkb);
        const int buf = lt & 1;
        if (lt >= 2) wait_cluster(&tempty[buf], ((lt >> 1) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t acc = tmem + buf * 256;
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % kPS;
          ptx::mbar_wait(&full[s], (it / kPS) & 1);
          wait_cluster(&pfull[s], (it / kPS) & 1);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + s * kPStage), sb = sa + kHalf;
#pragma unroll
          for (int k = 0; k < kGemmBlockK / 16; ++k)
            mma_pair(acc, ptx::umma_desc_sw128(sa + k * 2048, 8192, 1024), ptx::umma_desc_sw128(sb + k * 2048, 8192, 1024),
                     kIdesc, (i > 0 || k > 0) ? 1u : 0u);
          commit_pair(&empty[s]);
        }
        commit_pair(&tfull[buf]);
      }
    } else if (lane == 0) {
      // ---------------- forwarder (peer): its half of stage s landed -> leader's pfull[s]
      int it = 0;
      for (int t = cid; t < ntile; t += ncl) {
        int prob, split, kb0, nkb;
        decode(t, prob, split, kb0, nkb);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % kPS;
          ptx::mbar_wait(&full[s], (it / kPS) & 1);
          arrive_remote(&pfull[s], 0);
        }
      }
    }
  } else if (warp < 2 + kPEpiWarps) {
    // ---------------- epilogue: this CTA's 128 output rows x 256 columns -> fp32 slab
    constexpr int W = kPEpiWarps / 4;
    const int e = warp - 2, q = warp & 3, h = e >> 2;
    uint8_t* stage_base = staging + e * kPStaging;
    int lt = 0;
    for (int t = cid; t < ntile; t += ncl, ++lt) {
      int prob, split, kb0, nkb;
      decode(t, prob, split, kb0, nkb);
      const GemmProblem& pr = P.prob[prob];
      const int buf = lt & 1;
      const int rbase = int(rank) * 128 + q * 32;
      ptx::mbar_wait_sleep(&tfull[buf], (lt >> 1) & 1);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int c = h; c < 8; c += W) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(q * 32) << 16) + buf * 256 + c * 32, r);
        ptx::tmem_ld_wait();
        if (nkb == 0) {
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = 0u;
        }
        uint8_t* st = stage_base;
        if (lane == 0) ptx::bulk_wait_read<0>();
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(st + lane * 128 + ((j ^ (lane & 7)) << 4)) =
              make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          ptx::tma_store_3d(&pr.map_out, st, c * 32, rbase, split);
          ptx::bulk_commit();
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0)
          ptx::mbar_arrive(&tempty[buf]);
        else
          arrive_remote(&tempty[buf], 0);
      }
    }
    if (lane == 0) ptx::bulk_wait<0>();
  } else {
    // ---------------- column sums of this CTA's dPre half (bias gradient) while the MMA runs
    const int c = (warp - 2 - kPEpiWarps) * 32 + lane;  // 0..127
    const int box = c >> 6, cc = c & 63;
    int it = 0;
    for (int t = cid; t < ntile; t += ncl) {
      int prob, split, kb0, nkb;
      decode(t, prob, split, kb0, nkb);
      const GemmProblem& pr = P.prob[prob];
      const bool on = pr.colsum != nullptr;
      float sum = 0.f;
      for (int i = 0; i < nkb; ++i, ++it) {
        const int st = it % kPS;
        ptx::mbar_wait(&full[st], (it / kPS) & 1);
        if (on) {
          const uint8_t* sa = smem + st * kPStage + box * 8192 + (cc & 7) * 2;
#pragma unroll 8
          for (int rr = 0; rr < kGemmBlockK; ++rr) {
            const uint16_t v = *reinterpret_cast<const uint16_t*>(sa + rr * 128 + ((((cc >> 3) ^ (rr & 7))) << 4));
            sum += __uint_as_float(uint32_t(v) << 16);
          }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[st]);
      }
      if (on) pr.colsum[(long long)split * pr.M + int(rank) * 128 + c] = sum;
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();  // both CTAs done with the pair's TMEM and barriers
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

}  // namespace

// Pairs that can be resident at once (a CTA pair needs both SMs of a TPC; partitions and
// floorswept TPCs make this smaller than SMs / 2).
int gemm_pair_max_clusters() {
  static int n = -1;
  if (n < 0) {
    GMI_CUDA_CHECK(cudaFuncSetAttribute(gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * 256);
    cfg.blockDim = dim3(kPThreads);
    cfg.dynamicSmemBytes = kPSmem;
    GMI_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&n, gemm_pair_kernel, &cfg));
  }
  return n;
}

bool gemm_pair_applicable(int M, int N, int a_mn, int b_mn, int epi) {
  return M == 256 && N == 256 && a_mn == 1 && b_mn == 1 && epi == EPI_F32;
}

void gemm_pair_launch(const GemmParams& P, int max_ctas, cudaStream_t s) {
  for (int i = 0; i < P.num_problems; ++i)
    if (!gemm_pair_applicable(P.prob[i].M, P.prob[i].N, 1, 1, EPI_F32))
      invalid("SM-pair weight-gradient GEMM needs M = N = 256");
  static bool configured = false;
  if (!configured) {
    GMI_CUDA_CHECK(cudaFuncSetAttribute(gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem));
    configured = true;
  }
  const int tiles = P.num_problems * P.splits;
  const int clusters = std::max(1, std::min(tiles, (max_ctas > 0 ? max_ctas : device_sm_count()) / 2));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = kPSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GMI_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gemm_pair_kernel, P));
}

}  // namespace gmi

extern "C" GMI_API int gmi_dev_pair_clusters(int* out) {
  return gmi::guarded([&] {
    if (!out) gmi::invalid("null argument");
    *out = gmi::gemm_pair_max_clusters();
  });
}
