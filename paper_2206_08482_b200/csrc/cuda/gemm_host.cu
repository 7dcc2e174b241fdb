// Host side of the tcgen05 GEMM: TMA tensor-map encoding, tile-count based block-N choice,
// template dispatch, and a C-ABI diagnostic entry point used by the GPU parity tests.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "../host/errors.hpp"
#include "gemm.cuh"
#include "gemm_host.hpp"

namespace gmi {

namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) fail(GMI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  return fn;
}

CUtensorMap encode(CUtensorMapDataType dt, int rank, const void* base, const cuuint64_t* dims,
                   const cuuint64_t* strides_bytes, const cuuint32_t* box, CUtensorMapSwizzle sw) {
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) invalid("TMA base address must be 16-byte aligned");
  for (int i = 0; i < rank - 1; ++i)
    if (strides_bytes[i] % 16 != 0) invalid("TMA row pitch must be a multiple of 16 bytes");
  CUtensorMap map;
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&map, dt, cuuint32_t(rank), const_cast<void*>(base), dims, strides_bytes, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(GMI_ERR_CUDA, "cuTensorMapEncodeTiled failed with code " + std::to_string(int(r)));
  return map;
}

}  // namespace

CUtensorMap make_tma_2d_bf16(const void* base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                             uint32_t box_outer) {
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  return encode(CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

CUtensorMap make_tma_out_bf16(const void* base, uint64_t cols, uint64_t rows, uint64_t ld) {
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {32, 32};
  return encode(CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B);
}

CUtensorMap make_tma_out_f32(const void* base, uint64_t cols, uint64_t rows, uint64_t splits, uint64_t ld,
                             uint64_t split_stride) {
  const cuuint64_t dims[3] = {cols, rows, splits};
  const cuuint64_t strides[2] = {ld * 4, split_stride * 4};
  const cuuint32_t box[3] = {32, 32, 1};
  return encode(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

CUtensorMap tma_kmajor(const void* p, int cols, long long rows, long long ld, int box_rows) {
  return make_tma_2d_bf16(p, uint64_t(cols), uint64_t(rows), uint64_t(ld), kGemmBlockK, uint32_t(box_rows));
}

CUtensorMap tma_aux(const void* p, int cols, long long rows, long long ld) {
  return make_tma_2d_bf16(p, uint64_t(cols), uint64_t(rows), uint64_t(ld), 64, kGemmBlockM);
}

CUtensorMap tma_mnmajor(const void* p, int cols, long long rows, long long ld) {
  return make_tma_2d_bf16(p, uint64_t(cols), uint64_t(rows), uint64_t(ld), 64, 64);
}

int device_sm_count() {
  int dev = 0, n = 0;
  GMI_CUDA_CHECK(cudaGetDevice(&dev));
  GMI_CUDA_CHECK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

int gemm_tiles(int M, int N, int bn, int problems, int splits) {
  return ((M + kGemmBlockM - 1) / kGemmBlockM) * ((N + bn - 1) / bn) * problems * splits;
}

int gemm_choose_bn(int M, int N, int problems, int splits, int sms) {
  const int cands[3] = {256, 128, 64};
  for (int bn : cands) {
    if (bn > ((N + 63) / 64) * 64) continue;
    if (gemm_tiles(M, N, bn, problems, splits) >= 4 * sms) return bn;
  }
  return 64;
}

namespace {

template <int BN, int AMN, int BMN, int EPI, int WS = 0, int CS = 0>
void launch_t(const GemmParams& P, int ctas, cudaStream_t s) {
  constexpr int smem = GemmSmem<BN, EPI, WS>::kBytes;
  auto kern = gemm_tcgen05_kernel<BN, AMN, BMN, EPI, WS, CS>;
  static bool configured = false;  // per instantiation
  if (!configured) {
    GMI_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  launch_pdl(kern, dim3(ctas), dim3(gemm_threads(EPI) + 128 * CS), smem, s, P);
}

template <int BN>
void launch_bn(const GemmParams& P, int a_mn, int b_mn, int epi, int ctas, cudaStream_t s, int ws) {
  const int key = a_mn * 100 + b_mn * 10 + epi;
  bool cs = false;
  for (int i = 0; i < P.num_problems; ++i) cs = cs || P.prob[i].colsum != nullptr;
  if (cs) {  // split-K weight gradient with fused bias-gradient column sums
    if (key != 1 * 100 + 1 * 10 + EPI_F32 || ws) invalid("column sums need the MN-major weight-gradient GEMM");
    return launch_t<BN, 1, 1, EPI_F32, 0, 1>(P, ctas, s);
  }
  if (ws == 2) {  // K <= 512 resident: block N <= 128 only (shared-memory budget)
    if constexpr (BN <= 128) {
      switch (key) {
        case 0 * 100 + 0 * 10 + EPI_BIAS_ELU: return launch_t<BN, 0, 0, EPI_BIAS_ELU, 2>(P, ctas, s);
        case 0 * 100 + 1 * 10 + EPI_DACT: return launch_t<BN, 0, 1, EPI_DACT, 2>(P, ctas, s);
        default: invalid("weight-stationary GEMM supports the forward and input-gradient epilogues only");
      }
    }
    invalid("weight-stationary GEMM with K > 256 needs block N <= 128");
  }
  if (ws) {
    switch (key) {
      case 0 * 100 + 0 * 10 + EPI_BIAS_ELU: return launch_t<BN, 0, 0, EPI_BIAS_ELU, 1>(P, ctas, s);
      case 0 * 100 + 1 * 10 + EPI_DACT: return launch_t<BN, 0, 1, EPI_DACT, 1>(P, ctas, s);
      default: invalid("weight-stationary GEMM supports the forward and input-gradient epilogues only");
    }
  }
  switch (key) {
    case 0 * 100 + 0 * 10 + EPI_BIAS_ELU: return launch_t<BN, 0, 0, EPI_BIAS_ELU>(P, ctas, s);
    case 0 * 100 + 0 * 10 + EPI_F32: return launch_t<BN, 0, 0, EPI_F32>(P, ctas, s);
    case 0 * 100 + 0 * 10 + EPI_DACT: return launch_t<BN, 0, 0, EPI_DACT>(P, ctas, s);
    case 0 * 100 + 1 * 10 + EPI_DACT: return launch_t<BN, 0, 1, EPI_DACT>(P, ctas, s);
    case 0 * 100 + 1 * 10 + EPI_F32: return launch_t<BN, 0, 1, EPI_F32>(P, ctas, s);
    case 1 * 100 + 1 * 10 + EPI_F32: return launch_t<BN, 1, 1, EPI_F32>(P, ctas, s);
    case 1 * 100 + 0 * 10 + EPI_F32: return launch_t<BN, 1, 0, EPI_F32>(P, ctas, s);
    default: invalid("unsupported GEMM operand-major / epilogue combination");
  }
}

}  // namespace

int gemm_ws_bn(int M, int N, int K, int problems, int sms) {
  const int bn = N <= 64 ? 64 : N <= 128 ? 128 : 256;  // instantiated block widths
  if (N > 256 || K > kGemmMaxKbWS * kGemmBlockK) return 0;
  if (((M + kGemmBlockM - 1) / kGemmBlockM) * problems < sms) return 0;
  return bn;
}

int gemm_ws_wide(int M, int N, int K, int nets, int sms, int* parts) {
  const int np = (N + 127) / 128;
  if (K > gemm_ws_kb(2) * kGemmBlockK || nets * np > kGemmMaxProblems) return 0;
  if (((M + kGemmBlockM - 1) / kGemmBlockM) * nets * np < sms) return 0;
  *parts = np;
  return K <= kGemmMaxKbWS * kGemmBlockK ? 1 : 2;
}

int gemm_ws_grid(int M, int problems, int max_ctas) {
  const int tiles = ((M + kGemmBlockM - 1) / kGemmBlockM) * problems;
  const int ctas = std::max(1, std::min(tiles, max_ctas > 0 ? max_ctas : device_sm_count()));
  return std::max(problems, ctas / problems * problems);  // one problem per CTA
}

void gemm_launch(const GemmParams& P, int bn, int a_mn, int b_mn, int epi, cudaStream_t s, int max_ctas, int ws) {
  static int sms = 0;
  if (!sms) sms = device_sm_count();
  // weight-stationary problems (one per CTA) may differ in N (<= block N): a layer split into
  // 128-column parts has a narrower last part
  // (also split-K groups whose problems each fit one block N: the tile schedule is then the
  // same for all of them, e.g. every layer's weight gradient in one launch)
  const bool one_ntile = P.prob[0].N <= bn;
  int tiles = 0;
  GemmParams Q;  // heterogeneous groups: P with the per-problem tile offsets filled in
  if (P.hetero) {  // own M, N per problem (split-K weight gradients of layers of different widths)
    if (ws || P.chain > 1) invalid("heterogeneous GEMM groups are split-K launches");
    Q = P;
    Q.tile0[0] = 0;
    for (int i = 0; i < P.num_problems; ++i) {
      if (P.prob[i].K != P.prob[0].K) invalid("grouped GEMM problems must share K");
      Q.tile0[i + 1] = Q.tile0[i] + gemm_tiles(P.prob[i].M, P.prob[i].N, bn, 1, P.splits);
    }
    tiles = Q.tile0[P.num_problems];
  } else {
    for (int i = 1; i < P.num_problems; ++i)
      if (P.prob[i].M != P.prob[0].M || (ws || one_ntile ? P.prob[i].N > bn : P.prob[i].N != P.prob[0].N) ||
          P.prob[i].K != P.prob[0].K)
        invalid("grouped GEMM problems must share M, N, K");
    tiles = gemm_tiles(P.prob[0].M, P.prob[0].N, bn, P.num_problems, P.splits);
  }
  int ctas = std::max(1, std::min(tiles, max_ctas > 0 ? max_ctas : sms));
  if (ws) {
    if (ws < 0 || ws > 2 || P.splits != 1 || P.prob[0].N > bn || P.prob[0].K > gemm_ws_kb(ws) * kGemmBlockK)
      invalid("weight-stationary GEMM needs splits == 1, N <= block_n, K <= 256 (ws = 1) / 512 (ws = 2)");
    ctas = gemm_ws_grid(P.prob[0].M, P.num_problems, max_ctas > 0 ? max_ctas : sms);
  }
  if (P.chain > 1) {  // chained forward layers: one grid shape for all of them
    if (ws != 1 || epi != EPI_BIAS_ELU || P.chain * P.num_problems > kGemmMaxProblems)
      invalid("chained GEMM: weight-stationary forward layers only, at most 8 problems in all");
    for (int i = 0; i < P.chain * P.num_problems; ++i)
      if (P.prob[i].M != P.prob[0].M || P.prob[i].N != bn || P.prob[i].K > kGemmMaxKbWS * kGemmBlockK)
        invalid("chained GEMM layers must share M and have N == block_n, K <= 256");
  }
  const GemmParams& PL = P.hetero ? Q : P;
  switch (bn) {
    case 64: return launch_bn<64>(PL, a_mn, b_mn, epi, ctas, s, ws);
    case 128: return launch_bn<128>(PL, a_mn, b_mn, epi, ctas, s, ws);
    case 256: return launch_bn<256>(PL, a_mn, b_mn, epi, ctas, s, ws);
    default: invalid("GEMM block_n must be 64, 128 or 256");
  }
}

}  // namespace gmi

extern "C" GMI_API int gmi_dev_gemm(int a_mn, int b_mn, int epi, int M, int N, int K, const void* A, long long lda,
                                    const void* B, long long ldb, void* out, long long ldo, const float* bias,
                                    const void* aux, long long ld_aux, int splits, int weight_stationary,
                                    void* stream) {
  return gmi::guarded([&] {
    if (M <= 0 || N <= 0 || K <= 0) gmi::invalid("gemm dims must be positive");
    if (N % 32 != 0) gmi::invalid("gemm N must be a multiple of 32");
    if (splits < 1) gmi::invalid("splits must be >= 1");
    const int bn = weight_stationary ? ((N + 63) / 64) * 64 : gmi::gemm_choose_bn(M, N, 1, splits, gmi::device_sm_count());
    gmi::GemmParams P{};
    gmi::GemmProblem& p = P.prob[0];
    p.map_a = a_mn ? gmi::tma_mnmajor(A, M, K, lda) : gmi::tma_kmajor(A, K, M, lda, gmi::kGemmBlockM);
    p.map_b = b_mn ? gmi::tma_mnmajor(B, N, K, ldb) : gmi::tma_kmajor(B, K, N, ldb, bn);
    p.map_out = epi == gmi::EPI_F32 ? gmi::make_tma_out_f32(out, N, M, splits, ldo, (uint64_t)M * ldo)
                                    : gmi::make_tma_out_bf16(out, N, M, ldo);
    p.M = M;
    p.N = N;
    p.K = K;
    const int nkb = (K + gmi::kGemmBlockK - 1) / gmi::kGemmBlockK;
    p.kb_per_split = (nkb + splits - 1) / splits;
    p.bias = bias;
    p.aux = static_cast<const __nv_bfloat16*>(aux);
    p.ld_aux = ld_aux;
    if (aux && epi == gmi::EPI_DACT && weight_stationary) p.map_aux = gmi::tma_aux(aux, N, M, ld_aux);
    P.num_problems = 1;
    P.splits = splits;
    gmi::gemm_launch(P, bn, a_mn, b_mn, epi, static_cast<cudaStream_t>(stream), 0, weight_stationary);
  });
}
